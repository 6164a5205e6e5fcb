mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
for i in 1 2; do for lib in paper_2503_08946_b200/libgespmm.so paper_2503_08946_b200/libgespmm_w2.so; do b=$(basename $lib .so)
GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --workload config4 --N 256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/w_c4n256_${b}_$i.log 2>&1
GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --workload config2 --N 256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/w_c2n256_${b}_$i.log 2>&1
done; done
