# round 2 (session 3), call 66: the 512-byte-row gather ring without warp barriers (each lane copies and
# reads only its own 16 bytes of a row; default build = nosync) vs with them (rsync); GPU suite and
# racecheck on the ring cases first
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c66_gputests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2_c66_gputests.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "(bit_exact_vs_twin and (128 or 256)) or (every_variant and ring) or schedules_bit_exact" > gpurun_out/r2_c66_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -n 3 gpurun_out/r2_c66_racecheck.log
b() { GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --steps ${3:-20} --workload $1 --op ${2:-sum} > gpurun_out/r2_c66_$1_${2:-sum}_${tag}_$i.json 2>>gpurun_out/r2_c66.err; echo "$tag $1 ${2:-sum} $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_c66_$1_${2:-sum}_${tag}_$i.json | head -1) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/r2_c66_$1_${2:-sum}_${tag}_$i.json | head -1)"; }
for i in 1 2; do
  for tag in nosync rsync; do
    if [ $tag = nosync ]; then unset GESPMM_LIB; else export GESPMM_LIB=paper_2503_08946_b200/libgespmm_$tag.so; fi
    b config4; b config4 max; b config4 mean; b config5 sum 10
  done
done
