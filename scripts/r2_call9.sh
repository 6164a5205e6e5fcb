# round 2, call 9: TMA gather4 ring on config 5's column stream, with and without per-gather4 L2 hints
set -x
timeout 900 python tools/l2hot_probe.py --tma 4:1:24,6:1:16,3:2:16,2:2:24 --hot-mb 64,96 > gpurun_out/r2_c9_tma.jsonl 2> gpurun_out/r2_c9_tma.err
tail -3 gpurun_out/r2_c9_tma.err
timeout 600 python tools/l2hot_probe.py --panels 128 --panel-u 0 --panel-modes 0 --ldgsts 4:4:4:24,4:8:2:24 --hot-mb 64 > gpurun_out/r2_c9_ring_ref.jsonl 2>&1
