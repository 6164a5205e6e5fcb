# round 2 (session 3), call 53: GPU suite on the build after the TMA experiment was taken out again
# (plan.last_variant diagnostics kept), and the config 5 / 4 kernel lines
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c53_gputests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2_c53_gputests.log
for w in config5 config4; do GESPMM_NO_PROBE=1 timeout 600 python bench.py --extra none --no-cpu-baseline --no-e2e --sustained-s 0 --workload $w > gpurun_out/r2_c53_$w.json 2>>gpurun_out/r2_c53.err; grep -o '"ms_per_step": [0-9.]*\|"kernel_variant": "[a-z0-9_]*"\|"build_ms": [0-9.]*\|"first_build_ms": [0-9.]*' gpurun_out/r2_c53_$w.json | head -5; done
