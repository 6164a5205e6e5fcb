# column-panel replay with an L2 hot set (tools/l2hot_probe.py --panels)
timeout 900 python tools/l2hot_probe.py --panels 32,64,128 --hot-mb 32,48,64,80 --panel-modes 0,1,2 > gpurun_out/r2_l2hot_panels.jsonl 2> gpurun_out/r2_l2hot_panels.err
timeout 1200 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:probe_w --csv --log-file gpurun_out/r2_l2hot_panels_ncu.csv python tools/l2hot_probe.py --panels 32,64,128 --hot-mb 48,64 --panel-modes 0,1 --reps 0 > gpurun_out/r2_l2hot_panels_ncu.jsonl 2>&1
