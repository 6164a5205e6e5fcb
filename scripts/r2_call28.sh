# round 2, call 28: 10,000-case fuzz with the one-shot entry point in every third case
GESPMM_FUZZ_CASES=10000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fuzz10000.log 2>&1; echo "fuzz rc=$?"
tail -3 gpurun_out/fuzz10000.log
