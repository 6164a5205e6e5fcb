# round 2 (session 3), call 43: paired-lane kernel at N=32/64/128 on the L1-pipe-bound config 3 (and configs 1/2)
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op ${3:-sum} ${2:+--variant $2} > gpurun_out/r2_c43_$1_${3:-sum}_${2:-default}_$i.json 2>>gpurun_out/r2_c43.err; echo "$1 ${3:-sum} ${2:-default} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c43_$1_${3:-sum}_${2:-default}_$i.json | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' gpurun_out/r2_c43_$1_${3:-sum}_${2:-default}_$i.json)"; }
for i in 1 2; do
  b config3-32; b config3-32 pair_vec2; b config3-32 "" max; b config3-32 pair_vec2 max
  b config3-64; b config3-64 pair_vec4
  b config3-128; b config3-128 pair_vec4
  b config1; b config1 pair_vec2
  b config2; b config2 pair_vec4
done
