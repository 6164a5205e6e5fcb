# round 2, call 27: whole-matrix bit-exactness at full size (configs 4, 5, 3-256) against the fp32 twin
set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k whole_matrix --durations=10 > gpurun_out/r2_c27_whole.log 2>&1; echo "pytest rc=$?"
tail -20 gpurun_out/r2_c27_whole.log
