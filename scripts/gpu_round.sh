# One GPU session: tests, full bench, comparison build, reference arm, launch list, full ncu.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.log 2>&1
for lib in paper_2503_08946_b200/libgespmm_*.so; do
  [ -e "$lib" ] || continue
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/bench_$b.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spmm_kernel|k_rows|k_count|k_emit|k_totals|k_colind|Scan" --csv --log-file gpurun_out/launches_${PROF_TAG:-x}.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 4 -c 1 -o gpurun_out/prof_${PROF_TAG:-x} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
