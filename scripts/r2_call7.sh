# round 2, call 7: hot-set register path with 8 rows per batch (tagged builds) vs the ring, configs 5 and 4
set -x
b() { timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps 10 --workload $1 > $2 2>>gpurun_out/r2_c7.err; echo "$2 $(grep -o '"ms_per_step": [0-9.]*' $2 | head -1)"; }
for w in config5 config4; do
  for i in 1 2; do
    GESPMM_HOT=0 b $w gpurun_out/r2_c7_${w}_ring_$i.json
    b $w gpurun_out/r2_c7_${w}_hotu4_$i.json
    for t in hu8b3 hu8b4 hu8b2; do GESPMM_LIB=paper_2503_08946_b200/libgespmm_$t.so b $w gpurun_out/r2_c7_${w}_${t}_$i.json; done
  done
done
