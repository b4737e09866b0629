# Scratch driver for one gpurun call (edited per experiment).
set -x
mkdir -p gpurun_out/deint
L=paper_1206_1187_b200/libbcnrand_b200.so
for r in 1 2; do
  for v in old new; do
    cp abtest/$v.so $L
    timeout 300 python tools/deint_perf.py 65,66,68,70,72,74,76,78,80,90,110,120 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $r, /" >> gpurun_out/deint/ab3.jsonl
  done
done
cp abtest/new.so $L
timeout 600 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "deinterleave or interleaved" 2>&1 | tail -3 > gpurun_out/deint/pytest.log
