# round 1 final: ncu --set full of the SpMM kernel on configs 2 (sum, max), 3 (N=64), 4, 5 and the launch list of the default bench command (profiles/r1_*_final_ncu.txt)
mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
prof() { tag=$1; w=$2; op=$3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${tag} -f python bench.py --workload $w --op $op --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ncu_${tag}.log 2>&1; }
prof c2sum config2 sum
prof c2max config2 max
prof c3_64 config3-64 sum
prof c4sum config4 sum
prof c5sum config5 sum
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/launches_bench.log 2>&1
