# round 2 (session 3), call 71: the paired-lane kernel's stage address through a shuffle
# (GESPMM_SPOS_SHFL_PAIR=1, default build = ps) vs recomputed per batch (nops)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op ${2:-sum} > gpurun_out/r2_c71_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c71.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c71_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in ps nops; do
    if [ $tag = ps ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config3-16; b config3-16 max; b config3-16 mean; b config3-32 max
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "16 or pair or 32" > gpurun_out/r2_c71_tests.log 2>&1; echo "tests rc=$?"; tail -n 1 gpurun_out/r2_c71_tests.log
