# round 2, call 15: e2e per-call spread on config 2 (host entry point) + device timeline
set -x
timeout 300 python tools/e2e_probe.py 20 > gpurun_out/r2_e2e_probe.txt 2>&1; cat gpurun_out/r2_e2e_probe.txt
bash scripts/gpu_e2e_timeline.sh; tail -25 gpurun_out/e2e_timeline.txt
