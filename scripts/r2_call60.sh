# round 2 (session 3), call 60: GPU suite + the 10,000-case fuzz on the build with the masked slow path
# (8-row batches), and kernel lines of the affected tiles
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c60_gputests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2_c60_gputests.log
GESPMM_FUZZ_CASES=10000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_c60_fuzz10000.log 2>&1; echo "fuzz rc=$?"; tail -n 1 gpurun_out/r2_c60_fuzz10000.log
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op ${2:-sum} > gpurun_out/r2_c60_$1_${2:-sum}.json 2>>gpurun_out/r2_c60.err; echo "$1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c60_$1_${2:-sum}.json | head -1)"; }
b config2; b config2 max; b config2 min; b config2 mean; b config3-32; b config3-64; b config1
