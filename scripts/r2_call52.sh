# round 2 (session 3), call 52: where the TMA ring loses -- hot set off (no bitmap lookup in the stage pass,
# every group evict_first) vs 80 MB hot set vs the cp.async ring; ncu of the TMA ring on config 4
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op ${2:-sum} > gpurun_out/r2_c52_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c52.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c52_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' gpurun_out/r2_c52_$1_${2:-sum}_${tag}_$i.json) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/r2_c52_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1; do
  for tag in tma tmanohot ring; do
    unset GESPMM_TMA GESPMM_HOT_ROWS
    [ $tag = ring ] && export GESPMM_TMA=0
    [ $tag = tmanohot ] && export GESPMM_HOT_ROWS=0
    b config4; b config5
  done
done
unset GESPMM_TMA GESPMM_HOT_ROWS
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 3 -c 1 \
    -o gpurun_out/prof_r2c52_tma_config4 -f python bench.py --workload config4 --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 --extra none > gpurun_out/ncu_r2c52.log 2>&1
