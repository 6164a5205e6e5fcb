# e2e diagnostics: bisect the host-path slowdown (untraced wall clock).
set -x
mkdir -p gpurun_out
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --soak-s 0.5 > gpurun_out/bench_e2e_$1.log 2>&1; }
run base
GESPMM_NO_SIDE_STREAM=1 run noside
GESPMM_NO_POOL_RESIDENT=1 run nopool
GESPMM_NO_SIDE_STREAM=1 GESPMM_NO_POOL_RESIDENT=1 run neither
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.json 2> gpurun_out/e2e_breakdown.err
