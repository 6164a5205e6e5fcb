# round 2 (session 4), call 78: config 5 / 4 at the 1000 W power cap -- the gather ring (default) vs the register
# path (GESPMM_RING=0), sustained leg with board power and SM clock, alternating twice
set -x
mkdir -p gpurun_out/r2_power
b() { GESPMM_RING=$3 GESPMM_NO_PROBE=1 timeout 600 python bench.py --workload $1 --op sum --steps 20 --warmup 5 --extra none --no-cpu-baseline --no-e2e --sustained-s 2 > gpurun_out/r2_power/$1_ring$3_$2.log 2>&1; python -c "
import json,sys
l=json.loads(open('gpurun_out/r2_power/$1_ring$3_$2.log').read().strip().splitlines()[-1])
print('$1 ring=$3 rep=$2', round(l['ms_per_step'],3), l['kernel_variant'], l['clocks']['sm_mhz'], 'sustained', round(l['sustained']['ms_per_step'],3), l['sustained']['clocks']['sm_mhz'], l['sustained']['clocks'].get('power_w'))"; }
for rep in 1 2; do b config5 $rep 1; b config5 $rep 0; done
for rep in 1 2; do b config4 $rep 1; b config4 $rep 0; done
