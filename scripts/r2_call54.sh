# round 2 (session 3), call 54: the stage window address produced by a shuffle (GESPMM_SPOS_SHFL=1, spos)
# so ptxas keeps it in a register instead of rematerializing it per batch, vs the default build
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c54_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c54.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c54_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in spos head; do
    if [ $tag = head ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config2; b config2 max; b config2 mean; b config3-32; b config3-64; b config3-256; b config4; b config4 max; b config5 sum 10
  done
done
