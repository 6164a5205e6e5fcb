# round 2 (session 4), call 77: the default line with board power (NVML power draw vs the enforced limit) in the
# timed-region clock record; bench GPU tests
set -x
mkdir -p gpurun_out/r2_power
timeout 900 python bench.py > gpurun_out/r2_power/default.log 2>&1; echo "default rc=$?"
timeout 600 python -m pytest tests/test_bench_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_power/pytest_bench.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_power/pytest_bench.log
