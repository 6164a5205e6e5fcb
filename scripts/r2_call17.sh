# round 2, call 17: pinned per-warp constants (GESPMM_PIN=1, current tree) vs the committed build (libgespmm_base.so)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${4:-20} --workload $1 --op $2 > $3 2>>gpurun_out/r2_c17.err; echo "$3 $(grep -o '"ms_per_step": [0-9.]*' $3 | head -1)"; }
for i in 1 2; do
  for w in "config2 sum" "config2 max" "config2 mean" "config3-16 sum" "config3-32 sum" "config3-64 sum" "config4 sum" "config4 mean" "config5 sum"; do
    set -- $w
    st=20; [ "$1" = "config5" ] && st=8
    b $1 $2 gpurun_out/r2_c17_$1_$2_new_$i.json $st
    GESPMM_LIB=paper_2503_08946_b200/libgespmm_base.so b $1 $2 gpurun_out/r2_c17_$1_$2_base_$i.json $st
  done
done
