# round 2 (session 3), call 57: row seeds behind a warp-uniform branch on the accumulate flag
# (GESPMM_SEED_BRANCH=1, default build = sb) vs the select form (nosb)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c57_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c57.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c57_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in sb nosb; do
    if [ $tag = sb ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config2; b config2 max; b config2 mean; b config1; b config3-32; b config3-64; b config4
  done
done
