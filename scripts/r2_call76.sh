# round 2 (session 4), call 76: compute-sanitizer (memcheck incl. the host pipeline's chunk-rule test, racecheck,
# synccheck) on the final build (the paired-lane shuffle change and the 64-chunk cap came after the last run)
set -x
bash scripts/gpu_sanitize.sh
tail -n 3 gpurun_out/san_memcheck.log gpurun_out/san_racecheck.log gpurun_out/san_synccheck.log
