# Full GPU tests, then the sweep of the BASELINE configs (kernel-only lines) + the default bench line.
mkdir -p gpurun_out/sweep
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --workload $1 --op $2 --steps ${3:-20} --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/sweep/$1_$2.log 2>&1; }
b config1 sum
for op in sum max min mean; do b config2 $op; done
for n in 16 32 64 128 256; do b config3-$n sum; done
for op in sum max min mean; do b config4 $op; done
for op in sum max; do b config5 $op 10; done
timeout 900 python bench.py > gpurun_out/sweep/default.log 2>&1
