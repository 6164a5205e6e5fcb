# round 2 (session 3), call 40: state check after the container restore -- GPU suite, smoke, default bench line
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_c40_gputests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_c40_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2_c40_default.json 2> gpurun_out/r2_c40_default.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_c40_gputests.log
