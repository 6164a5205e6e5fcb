# Full GPU tests, then every BASELINE config/op as a kernel-only bench line
# (clocks sampled in the timed region), then the default bench line.
mkdir -p gpurun_out/sweep
GESPMM_PARITY_OUT=gpurun_out/sweep/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --workload $1 --op $2 --steps ${3:-20} --warmup 5 --extra none --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/sweep/$1_$2.log 2>&1; echo "$1 $2 $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep/$1_$2.log | head -1)"; }
b config1 sum
for op in sum max min mean; do b config2 $op; done
for n in 16 32 64 128 256; do b config3-$n sum; done
for op in sum max min mean; do b config4 $op; done
for op in sum max min mean; do b config5 $op 10; done
timeout 900 python bench.py > gpurun_out/sweep/default.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/sweep/reference.log 2>&1; echo "reference rc=$?"
