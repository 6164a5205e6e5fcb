# One GPU session: tests, benches, ncu capture of the no-gather ablation.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for lib in paper_2503_08946_b200/libgespmm*.so; do
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/bench_$b.log 2>&1
done
GESPMM_LIB=$PWD/paper_2503_08946_b200/libgespmm_nogather.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 4 -c 1 -o gpurun_out/prof_nogather python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 4 -c 1 -o gpurun_out/prof_r1h python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
