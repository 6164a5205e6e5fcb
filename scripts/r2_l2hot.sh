# L2 hot-set probe on config 5's column stream (tools/l2hot_probe.py)
timeout 900 python tools/l2hot_probe.py > gpurun_out/r2_l2hot.jsonl 2> gpurun_out/r2_l2hot.err
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:probe_hot --csv --log-file gpurun_out/r2_l2hot_ncu.csv python tools/l2hot_probe.py --reps 0 --persist 0,max > gpurun_out/r2_l2hot_ncu.jsonl 2>&1
