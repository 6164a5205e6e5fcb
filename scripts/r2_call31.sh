# round 2, call 31: full GPU suite + 10,000-case fuzz on the U=12-sum build
set -x
GESPMM_PARITY_OUT=gpurun_out/r2_c31_parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_c31_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_c31_tests.log
GESPMM_FUZZ_CASES=10000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fuzz10000.log 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/fuzz10000.log
