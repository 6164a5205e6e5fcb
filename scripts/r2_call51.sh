# round 2 (session 3), call 51: TMA gather4 ring with the plan's L2 hot set -- parity tests, then config 5 / 4
# kernel A/B: auto (TMA) vs GESPMM_TMA=0 (cp.async ring, same library) vs HEAD's library (base)
set -x
timeout 300 python -m pytest tests/test_gpu_tma.py -x -q > gpurun_out/r2_c51_tma_tests.log 2>&1; rc=$?; echo "tma tests rc=$rc"; tail -n 15 gpurun_out/r2_c51_tma_tests.log
[ $rc -ne 0 ] && exit 1
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op ${2:-sum} > gpurun_out/r2_c51_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c51.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c51_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' gpurun_out/r2_c51_$1_${2:-sum}_${tag}_$i.json) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/r2_c51_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in tma ring base; do
    unset GESPMM_LIB GESPMM_TMA
    [ $tag = ring ] && export GESPMM_TMA=0
    [ $tag = base ] && export GESPMM_LIB=paper_2503_08946_b200/libgespmm_base.so
    b config5; b config4
  done
done
