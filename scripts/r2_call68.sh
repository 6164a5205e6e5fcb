# round 2 (session 3), call 68: register gathers with 8-row batches at 3 CTAs/SM (r8m3, GESPMM_RING=0:
# the ring's rows in flight without its shared-memory traffic) vs the gather ring (default), configs 5 / 4
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c68_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c68.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c68_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/r2_c68_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' gpurun_out/r2_c68_$1_${2:-sum}_${tag}_$i.json)"; }
for i in 1 2; do
  for tag in ring r8m3; do
    unset GESPMM_LIB GESPMM_RING
    [ $tag = r8m3 ] && export GESPMM_LIB=paper_2503_08946_b200/libgespmm_r8m3.so GESPMM_RING=0
    b config5 sum 10; b config4; b config4 max
  done
done
