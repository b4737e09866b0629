# Scratch driver for one gpurun call (edited per experiment).
set -x
mkdir -p gpurun_out/e2e
for r in 1 2; do for mb in 16 32 64 128 256 512; do
  BCN_HOST_CHUNK_MB=$mb timeout 300 python tools/e2e_chunk.py >> gpurun_out/e2e/chunk.jsonl 2>>gpurun_out/e2e/err.log
done; done
