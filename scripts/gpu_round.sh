# One GPU session: parity tests, bench (occupancy variants), ncu launch list + full capture.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for lib in libgespmm.so libgespmm_mb3.so libgespmm_mb5.so; do
  GESPMM_LIB=$PWD/paper_2503_08946_b200/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --soak-s 0.5 > gpurun_out/bench_$lib.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 --op max --no-cpu-baseline --no-e2e --soak-s 0.5 > gpurun_out/bench_max.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 4 -c 1 -o gpurun_out/prof_r1b python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
