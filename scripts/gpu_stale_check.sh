mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "stale_entries or host_entry" > gpurun_out/stale_fixed.log 2>&1
GESPMM_LIB=$PWD/paper_2503_08946_b200/libgespmm_nofix.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "stale_entries" > gpurun_out/stale_nofix.log 2>&1
