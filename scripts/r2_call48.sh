# round 2 (session 3), call 48: config 5's stream through the TMA gather4 ring with the stage's positions
# regrouped hot-first (per-group L2 hints), sustained (mean of the 2nd half of 30 back-to-back reps)
set -x
export GESPMM_PROBE_SUSTAINED=1
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 100 > gpurun_out/r2_c48_smi.csv &
SMI=$!
P="timeout 900 python tools/l2hot_probe.py --workload config5 --reps 30"
$P --tma 3:2:16,2:4:8,3:4:8 --hot-mb 64,80 --tma-mode 2 >> gpurun_out/r2_c48_probe.jsonl 2>>gpurun_out/r2_c48.err
$P --tma 3:2:16,3:4:8 --hot-mb 64,80 --tma-mode 3 >> gpurun_out/r2_c48_probe.jsonl 2>>gpurun_out/r2_c48.err
$P --tma 3:2:16 --hot-mb 64 --tma-mode 1 >> gpurun_out/r2_c48_probe.jsonl 2>>gpurun_out/r2_c48.err
$P --panels 128 --panel-u 0 --panel-modes 0 --ldgsts 4:8:2:24 --hot-mb 0 >> gpurun_out/r2_c48_probe.jsonl 2>>gpurun_out/r2_c48.err
kill $SMI
cat gpurun_out/r2_c48_probe.jsonl
