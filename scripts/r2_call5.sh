# round 2, call 5: hot set on/off A/B (bench, configs 5/4); TMA bulk-copy ring probes (config 5 with L2 hints, config 2)
set -x
b() { timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 10 --workload $1 > $2 2>>gpurun_out/r2_c5_ab.err; grep -o '"ms_per_step": [0-9.]*' $2 | head -1; }
for w in config5 config4; do
  for i in 1 2; do for h in 1 0; do GESPMM_HOT=$h b $w gpurun_out/r2_c5_ab_${w}_hot${h}_$i.json; done; done
done
timeout 600 python tools/l2hot_probe.py --panels 128 --panel-u 0 --panel-modes 0,1 --hot-mb 64 --bulk 4:8:2,4:16:2,4:8:4 > gpurun_out/r2_c5_bulk_c5.jsonl 2> gpurun_out/r2_c5_bulk_c5.err
tail -2 gpurun_out/r2_c5_bulk_c5.err
timeout 600 python tools/gather_probe.py > gpurun_out/r2_c5_gather_probe_c2.json 2> gpurun_out/r2_c5_gather_probe_c2.err
tail -2 gpurun_out/r2_c5_gather_probe_c2.err
