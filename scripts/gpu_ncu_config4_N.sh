mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
for n in 64 256; do
  timeout 900 ncu --set full --clock-control none -k regex:spmm_kernel -s 3 -c 1 -o gpurun_out/prof_c4n$n -f python bench.py --workload config4 --N $n --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ncu_c4n$n.log 2>&1
  timeout 600 python bench.py --workload config4 --N $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/b_c4n$n.log 2>&1
done
