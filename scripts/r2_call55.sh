# round 2 (session 3), call 55: the rowptr window read through a shuffle-produced shared address
# (GESPMM_RP_SHFL=1, default build = rp) vs the generic-pointer reads (norp)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c55_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c55.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c55_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in rp norp; do
    if [ $tag = rp ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config2; b config2 max; b config2 mean; b config1; b config3-16; b config3-32; b config3-64; b config4
  done
done
