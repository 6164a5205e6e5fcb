# round 2, call 29: the north star's "large R-MAT, N=64..256" range -- DRAM throughput (ncu) and bench time
# of configs 4 and 5 at N = 64, 128, 256 on the final kernel
set -x
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed"
for w in config4 config5; do for n in 64 128 256; do
  GESPMM_NO_PROBE=1 timeout 900 ncu --metrics $M --clock-control none -k regex:spmm_kernel -s 3 -c 1 --csv --log-file gpurun_out/r2_c29_ncu_${w}_N$n.csv \
    python bench.py --workload $w --N $n --steps 2 --warmup 3 --extra none --no-cpu-baseline --no-e2e --no-clocks --sustained-s 0 > /dev/null 2>&1
  GESPMM_NO_PROBE=1 timeout 900 python bench.py --workload $w --N $n --steps 10 --warmup 3 --extra none --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r2_c29_bench_${w}_N$n.json 2>/dev/null
  echo "$w N=$n $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c29_bench_${w}_N$n.json | head -1)"
done; done
