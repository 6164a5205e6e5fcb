# round 2, call 19: uniform full-tile flag alone (libgespmm_allok.so, "new" here = committed build)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${4:-20} --workload $1 --op $2 > $3 2>>gpurun_out/r2_c23.err; echo "$3 $(grep -o '"ms_per_step": [0-9.]*' $3 | head -1)"; }
for i in 1 2; do
  for w in "config2 sum" "config2 max" "config2 mean" "config3-32 sum" "config3-64 sum" "config4 sum" "config1 sum" "config3-128 sum"; do
    set -- $w
    b $1 $2 gpurun_out/r2_c23_$1_$2_head_$i.json
    GESPMM_LIB=paper_2503_08946_b200/libgespmm_allok.so b $1 $2 gpurun_out/r2_c23_$1_$2_allok_$i.json
  done
done
