# deep LDGSTS rings (smem landing zone: more rows in flight than registers allow)
P="python tools/l2hot_probe.py --panel-u 0 --panels"
timeout 600 $P 64,128 --hot-mb 48,64 --panel-modes 0,1 --ldgsts 2:8:4:24,2:8:3:32,2:16:2:24,2:8:4:16,4:4:4:24,4:8:2:24,4:4:6:16,4:4:4:32 > gpurun_out/r2_ldgsts.jsonl 2>&1
