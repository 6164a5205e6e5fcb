# round 2 (session 3), call 58: the slow path (row-crossing batches) folded by row runs under a position
# bit mask (GESPMM_SLOW_MASK=1, default build = mask) vs the per-position compare-and-branch chain (nomask);
# GPU parity suite on the mask build first
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c58_gputests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2_c58_gputests.log
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c58_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c58.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c58_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in mask nomask; do
    if [ $tag = mask ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config2; b config2 max; b config2 mean; b config1; b config3-32; b config3-64; b config3-256; b config4; b config4 max; b config5 sum 10
  done
done
