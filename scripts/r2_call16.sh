# round 2, call 16: PCIe 2-D copy probe (profiles/r2_pcie_2d.jsonl) and the C++ host / sharded / comm_wait / invalid-CSR GPU tests
set -x
timeout 300 python tools/pcie_2d_probe.py > gpurun_out/r2_pcie_2d.jsonl 2>&1; cat gpurun_out/r2_pcie_2d.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cpp_host or sharded or comm_wait or invalid_csr" > gpurun_out/r2_c16_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_c16_tests.log
