# round 2, call 30: more rows in flight at the 64-column tile -- U=12 at 4 CTAs/SM (small spill), U=12 / U=16 at 3 CTAs/SM
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${4:-20} --workload $1 --op $2 --N ${5:-0} > $3 2>>gpurun_out/r2_c30.err; echo "$3 $(grep -o '"ms_per_step": [0-9.]*' $3 | head -1)"; }
for i in 1 2; do
  for w in "config2 sum" "config2 max" "config3-64 sum" "config4 sum 10 64" "config5 sum 5 64"; do
    set -- $w
    b $1 $2 gpurun_out/r2_c30_$1_$2_N${4:-x}_head_$i.json ${3:-20} ${4:-0}
    for t in u12 u12b3 u16b3; do GESPMM_LIB=paper_2503_08946_b200/libgespmm_$t.so b $1 $2 gpurun_out/r2_c30_$1_$2_N${4:-x}_${t}_$i.json ${3:-20} ${4:-0}; done
  done
done
