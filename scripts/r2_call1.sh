# round 2, call 1: GPU test suite, config-5 L2 hot-set probes, config-5 bench
set -x
free -g | head -2; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
GESPMM_PARITY_OUT=gpurun_out/r2_parity.jsonl timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_gputests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputests.log
timeout 900 python tools/l2hot_probe.py --hot-mb 32,48,64,80,96 > gpurun_out/r2_l2hot.jsonl 2> gpurun_out/r2_l2hot.err
timeout 900 python tools/l2hot_probe.py --panels 32,64,128 --hot-mb 32,48,64,80 --panel-modes 0,1,2 > gpurun_out/r2_l2hot_panels.jsonl 2> gpurun_out/r2_l2hot_panels.err
timeout 900 python bench.py --workload config5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r2_c5.json 2> gpurun_out/r2_c5.err
tail -3 gpurun_out/r2_c5.err
