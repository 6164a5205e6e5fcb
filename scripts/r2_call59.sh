# round 2 (session 3), call 59: masked slow path at 12-row (mask, default) vs 8-row sum batches at the
# 64-column tile (mu8: no spills) vs the per-position slow path at 12 rows (nomask)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op sum ${2:+--N $2} > gpurun_out/r2_c59_$1_N${2:-x}_${tag}_$i.json 2>>gpurun_out/r2_c59.err; echo "$tag $1 N${2:-x} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c59_$1_N${2:-x}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in mask mu8 nomask; do
    if [ $tag = mask ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config2; b config3-64; b config3-128; b config3-256; b config4 64; b config5 64 10
  done
done
