# round 2 (session 3), call 69 (as call 62, final build after the ITEM32 / ring changes): ncu --set full on the bench line's workloads and the
# sweep's other captured ones (one launch each), and the launch list of the default bench command
set -x
export GESPMM_NO_PROBE=1
prof() { tag=$1; w=$2; op=$3
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm -s 3 -c 1 \
    -o gpurun_out/prof_r2g_${tag} -f python bench.py --workload $w --op $op --steps 2 --warmup 3 --extra none \
    --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ncu_r2g_${tag}.log 2>&1; echo "prof $tag rc=$?"; }
prof c5sum config5 sum
prof c4sum config4 sum
prof c2sum config2 sum
prof c2max config2 max
prof c3_64 config3-64 sum
prof c3_16 config3-16 sum
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r2g_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/r2g_launches_bench.log 2>&1; echo "launches rc=$?"
