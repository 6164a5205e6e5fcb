# One GPU session: parity tests, experiment builds, e2e breakdown.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for lib in paper_2503_08946_b200/libgespmm*.so; do
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/bench_$b.log 2>&1
done
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.json 2> gpurun_out/e2e_breakdown.err
ls -la gpurun_out
