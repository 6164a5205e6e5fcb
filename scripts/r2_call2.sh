# round 2, call 2: the new default bench line (config 5 + config 2 extra), the reference arm, the N>1 bench tests
set -x
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "bench rc=$?"
tail -5 gpurun_out/r2_bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"
tail -5 gpurun_out/r2_bench_ref.err
timeout 900 python -m pytest tests/test_bench_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2_benchtests.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_benchtests.log
