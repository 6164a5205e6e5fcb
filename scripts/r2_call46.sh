# round 2 (session 3), call 46: sanitizers and the 10,000-case fuzz on the build with the new paired-lane
# stage permutation (and max/min at N=32 on the paired-lane kernel)
set -x
bash scripts/gpu_sanitize.sh
GESPMM_FUZZ_CASES=10000 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fuzz10000.log 2>&1; echo "fuzz rc=$?" >> gpurun_out/fuzz10000.log
tail -n 3 gpurun_out/san_memcheck.log gpurun_out/san_racecheck.log gpurun_out/san_synccheck.log gpurun_out/fuzz10000.log
