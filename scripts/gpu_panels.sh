mkdir -p gpurun_out
run() { w=$1; pw=$2; GESPMM_PANEL=$pw timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/pan_${w}_${pw}.log 2>&1; }
for pw in 0 64 128; do run config3-256 $pw; done
for pw in 0 64; do run config3-128 $pw; done
for pw in 0 32 64; do run config4 $pw; done
for pw in 0 32; do run config2 $pw; done
