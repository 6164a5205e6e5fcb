# round 2, call 4: full GPU suite (incl. the L2 hot-set parity tests), hot set on/off A/B on configs 4/5,
# ncu DRAM bytes + L2 hit of the config-5 kernel with the hot set, plan timings
set -x
GESPMM_PARITY_OUT=gpurun_out/r2_c4_parity.jsonl timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_c4_tests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_c4_tests.log
B="python bench.py --extra '' --no-cpu-baseline --no-e2e --sustained-s 0 --steps 10"
for w in config5 config4; do
  for h in 1 0 1 0; do GESPMM_HOT=$h timeout 600 $B --workload $w > gpurun_out/r2_c4_ab_${w}_hot$h.json 2>>gpurun_out/r2_c4_ab.err; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c4_ab_${w}_hot$h.json; done
done
for h in 1 0; do
GESPMM_HOT=$h timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmm_kernel -c 1 --csv --log-file gpurun_out/r2_c4_ncu_c5_hot$h.csv python bench.py --extra '' --no-cpu-baseline --no-e2e --sustained-s 0 --steps 1 --warmup 0 --no-clocks > /dev/null 2>&1
done
GESPMM_TRACE=3 timeout 300 python tools/plan_timing.py > gpurun_out/r2_c4_plan_timing.json 2> gpurun_out/r2_c4_plan_timing.err
cat gpurun_out/r2_c4_plan_timing.json
