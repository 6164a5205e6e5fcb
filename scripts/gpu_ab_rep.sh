# Repeated A/B (kernel only), libs interleaved: bash scripts/gpu_ab_rep.sh REPS workload:op ...
mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
reps=$1; shift
for i in $(seq 1 $reps); do for wo in "$@"; do
w=${wo%%:*}; op=${wo##*:}
for lib in paper_2503_08946_b200/libgespmm*.so; do
  b=$(basename $lib .so)
  GESPMM_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --op $op --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks --soak-s 0 --sustained-s 0 > gpurun_out/rep_${w}_${op}_${b}_$i.log 2>&1
done; done; done
