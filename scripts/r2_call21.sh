# round 2, call 21: ncu --set full of the pinned build (configs 5, 2, 3-64, 4)
mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
prof() { tag=$1; w=$2; op=$3
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${tag} -f python bench.py --workload $w --op $op --steps 2 --warmup 3 --extra none \
    --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/ncu_${tag}.log 2>&1; echo "prof $tag rc=$?"; }
prof r2p_c5sum config5 sum
prof r2p_c2sum config2 sum
prof r2p_c2max config2 max
prof r2p_c4sum config4 sum
prof r2p_c3_64 config3-64 sum
