# round 2, call 13: compute-sanitizer (memcheck incl. the one-shot async plan, invalid CSR and the
# panelled sharded path; racecheck; synccheck) and a 10,000-case fuzz on the round-2 build
set -x
bash scripts/gpu_sanitize.sh
tail -3 gpurun_out/san_memcheck.log gpurun_out/san_racecheck.log gpurun_out/san_synccheck.log
GESPMM_FUZZ_CASES=10000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fuzz10000.log 2>&1; echo "fuzz rc=$?"
tail -3 gpurun_out/fuzz10000.log
