# round 2, probe: the GPU box itself (memory, cores, SM clock, L2 size, SM count)
set -x
free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p.L2_cache_size, p.multi_processor_count)"
python - <<'PY'
import ctypes
c=ctypes.CDLL('libcudart.so') if False else None
PY
timeout 600 python bench.py --workload config5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/r2_probe_c5.json 2> gpurun_out/r2_probe_c5.err
tail -3 gpurun_out/r2_probe_c5.err
