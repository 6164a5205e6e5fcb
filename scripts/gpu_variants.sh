# Bench every built libgespmm*.so on config 2 (kernel only), then the default lib on other configs.
mkdir -p gpurun_out
for lib in paper_2503_08946_b200/libgespmm*.so; do
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/var_${b}.log 2>&1
done
for w in config4 config3-16 config3-64 config3-256; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/cfg_${w}.log 2>&1
done
