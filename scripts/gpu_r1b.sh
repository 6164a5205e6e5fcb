mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_graphgen.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_graphgen.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "full_size_configs" > gpurun_out/pytest_fullsize.log 2>&1
timeout 600 python bench.py --workload config5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --soak-s 0.5 > gpurun_out/b_config5.log 2>&1
timeout 600 python bench.py --workload config2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/b_config2.log 2>&1
timeout 600 python bench.py --workload config4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/b_config4.log 2>&1
