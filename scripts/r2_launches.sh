# launch list of the default bench command (cold, serialized under ncu): the SpMM kernel's share of a step
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/r2_launches_bench.log 2>&1; echo "launches rc=$?"
