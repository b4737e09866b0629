# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/u32tile
mkdir -p $F
L=paper_1206_1187_b200/libbcnrand_b200.so
r=0
for v in old new new old old new; do
  r=$((r+1))
  cp abtest/$v.so $L
  timeout 300 python tools/deint_perf.py 1,2,3,7,16,33,64,65,80,100,120,128 | grep '"itemsize": 4' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $r, /" >> $F/ab.jsonl
done
cp abtest/new.so $L
timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "deinterleave or interleaved" 2>&1 | tail -3 > $F/pytest.log
