# round 2, call 6: config-5 hot set through the cp.async ring: .ca + L2 hint, and a pinned hot set (prefetch evict_last + demote)
set -x
P="python tools/l2hot_probe.py --panels 128 --panel-u 0"
timeout 300 $P --panel-modes 0,2 --hot-mb 64 --ldgsts 4:4:4:24,4:8:2:24 > gpurun_out/r2_c6_ca_hint.jsonl 2> gpurun_out/r2_c6_ca_hint.err
tail -2 gpurun_out/r2_c6_ca_hint.err
timeout 600 python tools/l2hot_probe.py --pinned 8:2:24,4:4:24 --hot-mb 32,64,96 > gpurun_out/r2_c6_pinned.jsonl 2> gpurun_out/r2_c6_pinned.err
tail -2 gpurun_out/r2_c6_pinned.err
timeout 300 python tools/plan_timing.py > gpurun_out/r2_c6_plan_timing.json 2>&1
