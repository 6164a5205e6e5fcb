# more rows in flight: register replay with U=16/32, and the cp.async.bulk ring
P="python tools/l2hot_probe.py --panels"
timeout 300 $P 64 --hot-mb 48,64 --panel-modes 0,1 --panel-u 16 > gpurun_out/r2_mlp.jsonl 2>&1
timeout 300 $P 32 --hot-mb 64 --panel-modes 0,1 --panel-u 32 >> gpurun_out/r2_mlp.jsonl 2>&1
timeout 300 $P 128 --hot-mb 48 --panel-modes 0,1 --panel-u 16 >> gpurun_out/r2_mlp.jsonl 2>&1
timeout 600 $P 64,128 --hot-mb 48,64 --panel-modes 0,1 --panel-u 0 --bulk 2:16:2,2:16:4,2:32:2,4:8:4,4:16:2,4:8:2 >> gpurun_out/r2_mlp.jsonl 2>&1
