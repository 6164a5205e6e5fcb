# round 2, call 26: column-panel width re-check on the final kernel (config 3, N=128/256) + the default line with extras
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 > $2 2>>gpurun_out/r2_c26.err; echo "$2 $(grep -o '"ms_per_step": [0-9.]*' $2 | head -1)"; }
for i in 1 2; do
  for p in 64 128 32; do GESPMM_PANEL=$p b config3-256 gpurun_out/r2_c26_c3-256_p${p}_$i.json; done
  for p in 64 0; do GESPMM_PANEL=$p b config3-128 gpurun_out/r2_c26_c3-128_p${p}_$i.json; done
done
timeout 900 python bench.py > gpurun_out/r2_c26_default.json 2> gpurun_out/r2_c26_default.err; echo "default rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2_c26_default.json'));print({k:(v.get('ms_per_step'),v.get('clocks',{}) and v['clocks'].get('sm_mhz')) for k,v in d['extra'].items()})"
