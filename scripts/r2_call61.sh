# round 2 (session 3), call 61: gather ring with 8-row batches at 2 CTAs/SM (ru8) vs 4-row batches at
# 3 CTAs/SM (default) for the 512-byte rows (configs 4/5)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c61_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c61.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c61_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/r2_c61_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in ru4 ru8; do
    if [ $tag = ru4 ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config4; b config4 max; b config4 mean; b config5 sum 10
  done
done
