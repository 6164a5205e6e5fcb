# round 2 (session 3), call 64: 32-bit item cursor (GESPMM_ITEM32=1, default build = i32) vs 64-bit (i64):
# fewer registers live across an item (vec2 spills 40/88 -> 24/40 bytes)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c64_gputests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2_c64_gputests.log
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c64_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c64.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c64_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in i32 i64; do
    if [ $tag = i32 ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config2; b config2 max; b config2 mean; b config1; b config3-16; b config3-32; b config3-64; b config4; b config5 sum 10
  done
done
