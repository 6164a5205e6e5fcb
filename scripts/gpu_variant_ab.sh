# Variant A/B (kernel only): bash scripts/gpu_variant_ab.sh workload:op:variant ...
mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
for wov in "$@"; do
IFS=: read w op v <<< "$wov"
timeout 300 python bench.py --workload $w --op $op --variant "$v" --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/var_${w}_${op}_${v:-auto}.log 2>&1
done
