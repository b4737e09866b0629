# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/pitch
mkdir -p $F
L=paper_1206_1187_b200/libbcnrand_b200.so
for r in 1 2; do
  for v in old new; do
    cp abtest/$v.so $L
    timeout 300 python tools/deint_perf.py 2,3,5,7,9,12,16,24 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $r, /" >> $F/ab.jsonl
  done
done
cp abtest/new.so $L
timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "deinterleave or interleaved" 2>&1 | tail -3 > $F/pytest.log
