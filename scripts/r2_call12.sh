# round 2, call 12: best case of a per-gather4 L2 hint -- TMA gather4 ring on config 5's stream with
# each span's hot positions gathered first (pure hot / cold groups)
set -x
timeout 900 python tools/l2hot_probe.py --tma 3:2:16,2:2:24,6:1:16 --hot-mb 64,96 --tma-sorted > gpurun_out/r2_c12_tma_sorted.jsonl 2> gpurun_out/r2_c12_tma_sorted.err
tail -3 gpurun_out/r2_c12_tma_sorted.err
