# round 2 (session 3), call 72: the final record again after the paired-lane shuffle change -- GPU suite + every BASELINE
# config/op (scripts/gpu_sweep.sh, default line and the reference arm included) + the 10,000-case fuzz
set -x
bash scripts/gpu_sweep.sh
GESPMM_FUZZ_CASES=10000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fuzz10000.log 2>&1; echo "fuzz rc=$?"; tail -n 1 gpurun_out/fuzz10000.log
