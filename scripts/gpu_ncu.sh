# ncu --set full of the SpMM kernel on the given workloads: scripts/gpu_ncu.sh TAG WORKLOAD [WORKLOAD...]
mkdir -p gpurun_out
tag=$1; shift
for w in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${tag}_${w} -f python bench.py --workload $w --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ncu_${tag}_${w}.log 2>&1
done
for w in "$@"; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/cfg_${tag}_${w}.log 2>&1
done
