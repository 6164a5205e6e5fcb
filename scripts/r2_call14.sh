# round 2, call 14: gather ring depth 3 at 3 CTAs/SM (smaller tiles/stage make room) vs depth 2, configs 5/4
set -x
b() { timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 10 --workload $1 > $2 2>>gpurun_out/r2_c14.err; echo "$2 $(grep -o '"ms_per_step": [0-9.]*' $2 | head -1)"; }
for w in config5 config4; do
  for i in 1 2; do
    b $w gpurun_out/r2_c14_${w}_base_$i.json
    for t in rd3 rd2t112; do GESPMM_LIB=paper_2503_08946_b200/libgespmm_$t.so b $w gpurun_out/r2_c14_${w}_${t}_$i.json; done
  done
done
