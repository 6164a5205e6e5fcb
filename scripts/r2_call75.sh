# round 2 (session 4), call 75: kernel time with 16-byte-aligned colind/vals vs a 4-byte offset view (the 4-byte
# staging path a rank's row-block view took when its first nonzero p0 % 4 != 0), configs 5/4/2; sharded GPU tests
# after local_block / the bench copy shard slabs into their own storage
set -x
mkdir -p gpurun_out/r2_align
timeout 900 python tools/align_probe.py config5 config4 config2 > gpurun_out/r2_align/align.jsonl 2> gpurun_out/r2_align/align.err; echo "align rc=$?"; cat gpurun_out/r2_align/align.jsonl; tail -3 gpurun_out/r2_align/align.err
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "shard or nccl or peer or bench" > gpurun_out/r2_align/pytest_shard.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_align/pytest_shard.log
