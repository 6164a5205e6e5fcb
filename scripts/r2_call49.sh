# round 2 (session 3), call 49: as call 48 with the regrouping done warp-cooperatively (ballot + per-warp
# scratch; mode 4 = the grouping with no hints, its cost alone), sustained
set -x
export GESPMM_PROBE_SUSTAINED=1
P="timeout 900 python tools/l2hot_probe.py --workload config5 --reps 30"
for m in 4 2 3; do
  $P --tma 3:2:16,3:4:8 --hot-mb 64,80 --tma-mode $m >> gpurun_out/r2_c49_probe.jsonl 2>>gpurun_out/r2_c49.err
done
$P --tma 3:2:16 --hot-mb 64,80 --tma-mode 1 >> gpurun_out/r2_c49_probe.jsonl 2>>gpurun_out/r2_c49.err
cat gpurun_out/r2_c49_probe.jsonl
