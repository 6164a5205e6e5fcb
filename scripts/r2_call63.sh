# round 2 (session 3), call 63: final record of the round -- GPU suite + every BASELINE config/op
# (scripts/gpu_sweep.sh: default line and the reference arm included) and the launch list of the default
# bench command
set -x
bash scripts/gpu_sweep.sh
export GESPMM_NO_PROBE=1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r2f_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/r2f_launches_bench.log 2>&1; echo "launches rc=$?"
