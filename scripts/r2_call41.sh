# round 2 (session 3), call 41: ncu --set full of config 3 at N=16/32 (paired-lane / 1-column tiles),
# and the device timeline of config 5's e2e call (GESPMM_TRACE=3)
set -x
for w in config3-16 config3-32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 3 -c 1 \
    -o gpurun_out/prof_r2c41_${w} -f python bench.py --workload $w --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 --extra none > gpurun_out/ncu_r2c41_${w}.log 2>&1
done
GESPMM_TRACE=3 GESPMM_NO_PROBE=1 timeout 900 python bench.py --steps 3 --warmup 3 --extra none --no-cpu-baseline \
  --sustained-s 0 > gpurun_out/r2_c41_c5_e2e_trace.json 2> gpurun_out/r2_c41_c5_e2e_trace.err
echo done
