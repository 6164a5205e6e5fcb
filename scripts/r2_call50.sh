# round 2 (session 3), call 50: TMA gather4 ring at the shared-memory budget a kernel variant would have
# (stage + ring: 2 stages x 8 rows at 16 warps/SM) vs 3 stages, with / without the grouped hints; sustained
set -x
export GESPMM_PROBE_SUSTAINED=1
P="timeout 900 python tools/l2hot_probe.py --workload config5 --reps 30"
$P --tma 2:2:16,3:2:16,2:2:24 --hot-mb 64,80 --tma-mode 2 >> gpurun_out/r2_c50_probe.jsonl 2>>gpurun_out/r2_c50.err
cat gpurun_out/r2_c50_probe.jsonl
