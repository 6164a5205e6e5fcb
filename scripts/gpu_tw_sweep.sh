# Tile-work sweep (kernel only): bash scripts/gpu_tw_sweep.sh workload:op ...
mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
for wo in "$@"; do
w=${wo%%:*}; op=${wo##*:}
for tw in 0 8 16 32 64 128 256; do
  timeout 300 python bench.py --workload $w --op $op --tile-work $tw --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/tw_${w}_${op}_${tw}.log 2>&1
done; done
