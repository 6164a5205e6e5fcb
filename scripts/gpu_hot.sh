mkdir -p gpurun_out
run() { w=$1; h=$2; GESPMM_LIB=$PWD/paper_2503_08946_b200/libgespmm_hot.so GESPMM_HOT_POPC=$h timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/hot_${w}_$h.log 2>&1; }
for h in 30 6 5 -1; do run config5 $h; done
for h in 30 7 6 5; do run config4 $h; done
for h in 30 9 8 7; do run config2 $h; done
