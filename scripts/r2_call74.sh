# round 2 (session 4), call 74: the final record on the final build (host chunk-rule switches, 64-chunk cap) --
# GPU suite + every BASELINE config/op (scripts/gpu_sweep.sh, default line and the reference arm included),
# smoke, and the 10,000-case fuzz
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
bash scripts/gpu_sweep.sh
GESPMM_FUZZ_CASES=10000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fuzz10000.log 2>&1; echo "fuzz rc=$?"; tail -n 1 gpurun_out/fuzz10000.log
