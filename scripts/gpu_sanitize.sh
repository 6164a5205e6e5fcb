# compute-sanitizer over small parity cases: memcheck (OOB / misaligned / illegal) and
# racecheck (shared-memory hazards of the CRC staging protocol and the gather ring)
mkdir -p gpurun_out
K="bit_exact_vs_twin or every_variant or schedules_bit_exact or column_panels or accumulate or empty_and_degenerate or misaligned or strided or fused_peer_stores or execute_rows or graph or invalid_csr or single_chunk or sharded_spmm_ex or chunk_rules or pipelined_chunks"
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider -k "$K or fuzz" > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "(bit_exact_vs_twin and (64 or 128 or 16 or 32)) or misaligned or maximum_number_all_bits" > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "bit_exact_vs_twin and (64 or 16 or 32)" > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.log
