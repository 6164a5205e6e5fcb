# round 2, call 18: woff pinned too (current tree) vs the committed pin build (libgespmm_base.so)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${4:-20} --workload $1 --op $2 > $3 2>>gpurun_out/r2_c18.err; echo "$3 $(grep -o '"ms_per_step": [0-9.]*' $3 | head -1)"; }
for i in 1 2; do
  for w in "config2 sum" "config2 max" "config2 mean" "config3-32 sum" "config3-64 sum" "config4 sum" "config4 mean" "config1 sum"; do
    set -- $w
    b $1 $2 gpurun_out/r2_c18_$1_$2_new_$i.json
    GESPMM_LIB=paper_2503_08946_b200/libgespmm_base.so b $1 $2 gpurun_out/r2_c18_$1_$2_base_$i.json
  done
done
