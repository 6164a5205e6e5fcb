# round 2 (session 3), call 42: L1 data-pipe cost of warp-uniform stage reads (tools/uniform_load_probe.cu),
# and the per-instruction shared/global wavefronts of config 2 (ncu --set full)
set -x
./tools/uniform_load_probe > gpurun_out/r2_c42_uniform_load.jsonl 2>&1
bash scripts/gpu_ncu.sh r2c42 config2
cat gpurun_out/r2_c42_uniform_load.jsonl
