# round 2 (session 3), call 47: config 5's column stream replayed back to back (sustained power state):
# TMA gather4 ring vs LDGSTS ring, mean of the second half of 40 reps, SM clock / power sampled alongside
set -x
export GESPMM_PROBE_SUSTAINED=1
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 100 > gpurun_out/r2_c47_smi.csv &
SMI=$!
for cfg in "--tma 3:2:16" "--tma 6:1:16" "--panels 128 --panel-u 0 --panel-modes 0 --ldgsts 4:8:2:24" "--panels 128 --panel-u 0 --panel-modes 0 --ldgsts 4:4:4:24" "--tma 3:2:16"; do
  echo "start $(date +%s.%N) $cfg" >> gpurun_out/r2_c47_times.txt
  timeout 600 python tools/l2hot_probe.py --workload config5 --hot-mb 0 --reps 40 $cfg >> gpurun_out/r2_c47_probe.jsonl 2>>gpurun_out/r2_c47.err
  echo "end $(date +%s.%N)" >> gpurun_out/r2_c47_times.txt
done
GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 2 --steps 40 > gpurun_out/r2_c47_config5.json 2>>gpurun_out/r2_c47.err
kill $SMI
cat gpurun_out/r2_c47_probe.jsonl
