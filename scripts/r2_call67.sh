# round 2 (session 3), call 67: register gathers (GESPMM_RING=0) vs the gather ring at the 128-column tile
# under the power cap (config 5) and at full clock (config 4)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c67_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c67.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c67_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/r2_c67_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' gpurun_out/r2_c67_$1_${2:-sum}_${tag}_$i.json)"; }
for i in 1 2; do
  for tag in ring reg; do
    if [ $tag = ring ]; then unset GESPMM_RING; else export GESPMM_RING=0; fi
    b config5 sum 10; b config4
  done
done
