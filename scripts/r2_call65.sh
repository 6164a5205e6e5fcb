# round 2 (session 3), call 65: sanitizers on the final kernel (masked slow path, shuffled shared addresses,
# 32-bit item cursor), and a 2-rank dry run of the N>1 bench path on one GPU (gloo) with config 2
set -x
bash scripts/gpu_sanitize.sh
tail -n 3 gpurun_out/san_memcheck.log gpurun_out/san_racecheck.log gpurun_out/san_synccheck.log
GESPMM_BENCH_BACKEND=gloo GESPMM_NO_PROBE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload config2 --steps 5 --warmup 3 \
  > gpurun_out/r2_c65_n2_gloo.json 2> gpurun_out/r2_c65_n2_gloo.err; echo "n2 rc=$?"
tail -c 1500 gpurun_out/r2_c65_n2_gloo.json
