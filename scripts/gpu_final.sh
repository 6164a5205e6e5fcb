# Round-end measurement record: GPU tests + sweep + default line (gpu_sweep.sh),
# the reference arm, ncu captures + launch list (gpu_profiles_final.sh).
bash scripts/gpu_sweep.sh
timeout 900 python bench.py --impl reference > gpurun_out/sweep/reference.log 2>&1
bash scripts/gpu_profiles_final.sh
