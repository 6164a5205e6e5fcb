mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
for i in 1 2; do for w in config4 config5 config2; do
for lib in paper_2503_08946_b200/libgespmm_sep.so paper_2503_08946_b200/libgespmm.so; do
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ab2_${w}_${b}_$i.log 2>&1
done; done; done
