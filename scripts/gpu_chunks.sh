mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1
for w in config2 config3-64 config3-16 config4; do
for lib in paper_2503_08946_b200/libgespmm*.so; do
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ch_${w}_${b}.log 2>&1
done; done
