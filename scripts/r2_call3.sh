# round 2, call 3: new C-ABI sharded tests + bench N>1 test; config-5 hot-set probes for the ring (LDGSTS) and register paths
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "sharded or comm_wait" tests/test_bench_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2_c3_tests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_c3_tests.log
P="python tools/l2hot_probe.py --panels 128 --panel-modes 0,1"
timeout 600 $P --hot-mb 48,64,80 --panel-u 8 --ldgsts 4:4:2:24,4:4:4:24,4:8:2:24 > gpurun_out/r2_c3_ring_hot.jsonl 2> gpurun_out/r2_c3_ring_hot.err
tail -3 gpurun_out/r2_c3_ring_hot.err
timeout 600 $P --hot-mb 64 --panel-u 4 > gpurun_out/r2_c3_reg_u4.jsonl 2>&1
