# Host-path A/B: GPU tests, device timeline, e2e bench lines (nnz-ordered vs row-ordered chunks)
mkdir -p gpurun_out
export GESPMM_NO_PROBE=1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
bash scripts/gpu_e2e_timeline.sh
for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/e2e_new_$i.log 2>&1
  GESPMM_HOST_ROW_ORDER=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/e2e_row_$i.log 2>&1
done
