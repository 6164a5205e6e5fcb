# round 2 (session 3), call 56: ncu --set full of the current build (configs 2 and 4) for the per-block
# instruction breakdown (tools/sass_blocks.py)
set -x
bash scripts/gpu_ncu.sh r2c56 config2 config4
