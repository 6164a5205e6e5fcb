# round 2, call 22: the gather ring at the 64-column tile (GESPMM_RING=2) on the pinned build
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op $2 > $3 2>>gpurun_out/r2_c22.err; echo "$3 $(grep -o '"ms_per_step": [0-9.]*' $3 | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' $3)"; }
for i in 1 2; do
  for w in "config2 sum" "config3-64 sum" "config3-128 sum"; do
    set -- $w
    b $1 $2 gpurun_out/r2_c22_$1_$2_reg_$i.json
    GESPMM_RING=2 b $1 $2 gpurun_out/r2_c22_$1_$2_ring_$i.json
  done
done
