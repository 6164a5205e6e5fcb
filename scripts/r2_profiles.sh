# Round-2 measurement record: ncu --set full of the SpMM kernel on the default line's workloads
# (config 5 headline, config 2 extra), the launch list of the default bench command, and the
# ncu stall tables of the gather-only bulk-copy vs LDGSTS rings (the negative result, DESIGN 8.1).
mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
prof() { tag=$1; w=$2; op=$3
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${tag} -f python bench.py --workload $w --op $op --steps 2 --warmup 3 --extra none \
    --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ncu_${tag}.log 2>&1; echo "prof $tag rc=$?"; }
prof r2_c5sum config5 sum
prof r2_c2sum config2 sum
prof r2_c2max config2 max
prof r2_c4sum config4 sum
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/r2_launches_bench.log 2>&1; echo "launches rc=$?"
unset GESPMM_NO_PROBE
timeout 900 ncu --set full --clock-control none -k regex:probe_bulk --launch-skip 14 -c 1 -o gpurun_out/prof_r2_bulk_u16d2_w24 -f \
  python tools/gather_probe.py > gpurun_out/ncu_r2_bulk.log 2>&1; echo "bulk rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:probe_ring --launch-skip 21 -c 1 -o gpurun_out/prof_r2_ring_u16d2_w24 -f \
  python tools/gather_probe.py > gpurun_out/ncu_r2_ring.log 2>&1; echo "ring rc=$?"
