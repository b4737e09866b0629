# Scratch driver for one gpurun call (edited per experiment).
set -x
mkdir -p gpurun_out/deint
for r in 1 2; do
  for v in 0 1 2; do
    BCN_U32_TILE=$v timeout 300 python tools/deint_perf.py 129,150,200,1000,5000,100003,1000003 | grep '"itemsize": 4' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $r, /" >> gpurun_out/deint/u32tile.jsonl
  done
done
