# round 2 (session 4), call 79: the ring's 4-row batches under the masked slow path (GESPMM_SLOW_MASK_U4=1,
# libgespmm_m4.so) vs the element-by-element slow path (libgespmm.so), configs 5/4; parity of the m4 build
set -x
mkdir -p gpurun_out/r2_m4
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps $4 --workload $1 --op $2 > $3 2>>gpurun_out/r2_m4/err.log; echo "$3 $(grep -o '"ms_per_step": [0-9.]*' $3 | head -1) $(grep -o '"sm_mhz": [0-9.]*' $3 | head -1)"; }
for i in 1 2; do
  for w in "config5 sum 10" "config5 max 10" "config4 sum 20" "config4 mean 20"; do
    set -- $w
    b $1 $2 gpurun_out/r2_m4/$1_$2_base_$i.json $3
    GESPMM_LIB=paper_2503_08946_b200/libgespmm_m4.so b $1 $2 gpurun_out/r2_m4/$1_$2_m4_$i.json $3
  done
done
GESPMM_LIB=paper_2503_08946_b200/libgespmm_m4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider -k "every_variant or bit_exact_vs_twin or ring or fuzz or full_size" > gpurun_out/r2_m4/pytest_m4.log 2>&1; echo "pytest m4 rc=$?"; tail -1 gpurun_out/r2_m4/pytest_m4.log
