# round 2, call 32: sum at the 64-column tile with 16-row batches (72-byte spill) vs 12 (head)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${4:-20} --workload $1 --op $2 --N ${5:-0} > $3 2>>gpurun_out/r2_c32.err; echo "$3 $(grep -o '"ms_per_step": [0-9.]*' $3 | head -1)"; }
for i in 1 2; do
  for w in "config2 sum" "config3-64 sum" "config4 sum 10 64" "config5 sum 5 64"; do
    set -- $w
    b $1 $2 gpurun_out/r2_c32_$1_$2_N${4:-x}_head_$i.json ${3:-20} ${4:-0}
    GESPMM_LIB=paper_2503_08946_b200/libgespmm_s16.so b $1 $2 gpurun_out/r2_c32_$1_$2_N${4:-x}_s16_$i.json ${3:-20} ${4:-0}
  done
done
