# round 2 (session 3), call 45: paired-lane batch of 32 positions at one column per lane (pu32) and a
# 24-position in-row fast batch at one column per lane (fb24) vs the default build
set -x
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 20 --workload $1 --op ${2:-sum} > gpurun_out/r2_c45_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c45.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c45_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"kernel_variant": "[a-z0-9_]*"' gpurun_out/r2_c45_$1_${2:-sum}_${tag}_$i.json)"; }
for i in 1 2; do
  for tag in new pu32 fb24; do
    if [ $tag = new ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config3-16; b config3-16 max; b config3-32; b config1
  done
done
