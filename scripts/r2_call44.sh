# round 2 (session 3), call 44: conflict-free stage permutation in the paired-lane kernel (lane-pair shfl swap)
# vs the lane-per-block permutation (libgespmm_base.so = HEAD a2dc0de); GPU suite on the new build
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c44_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_c44_gputests.log
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op ${3:-sum} ${2:+--variant $2} > gpurun_out/r2_c44_$1_${3:-sum}_${2:-default}_${tag}_$i.json 2>>gpurun_out/r2_c44.err; echo "$tag $1 ${3:-sum} ${2:-default} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c44_$1_${3:-sum}_${2:-default}_${tag}_$i.json | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' gpurun_out/r2_c44_$1_${3:-sum}_${2:-default}_${tag}_$i.json)"; }
for i in 1 2; do
  for tag in new base; do
    if [ $tag = base ]; then export GESPMM_LIB=paper_2503_08946_b200/libgespmm_base.so; else unset GESPMM_LIB; fi
    b config3-16; b config3-16 "" max; b config3-32 pair_vec2; b config3-32 pair_vec2 max; b config3-32
  done
done
