# round 2 (session 4), call 73: smoke + host-entry GPU tests on the equal-PCIe-byte chunk rule, and the
# e2e A/B of the chunk rules (equal rows x16 vs equal bytes) on configs 5, 4 and 2 with device timelines
set -x
mkdir -p gpurun_out/r2_chunks
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_chunks/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_chunks/smoke.log
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "host_entry" > gpurun_out/r2_chunks/pytest_host.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_chunks/pytest_host.log
for w in config5 config4 config2; do
  timeout 900 python tools/e2e_chunks_probe.py --workload $w --reps 6 --timeline > gpurun_out/r2_chunks/$w.jsonl 2> gpurun_out/r2_chunks/${w}_timeline.txt; echo "$w rc=$?"; cat gpurun_out/r2_chunks/$w.jsonl | cut -c1-200
done
