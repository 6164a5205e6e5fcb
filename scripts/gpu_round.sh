# One GPU session: quick parity check + bench grid over builds.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "every_variant or bit_exact_vs_twin" > gpurun_out/pytest_gpu.log 2>&1
for lib in paper_2503_08946_b200/libgespmm*.so; do
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/bench_${b}.log 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 --variant vec2_lpr32_cwm1 > gpurun_out/bench_vec2.log 2>&1
ls -la gpurun_out
