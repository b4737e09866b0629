# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/inter2
mkdir -p $F
L=paper_1206_1187_b200/libbcnrand_b200.so
for r in 1 2 3; do
  for v in old new; do
    cp abtest/$v.so $L
    timeout 300 python tools/inter_perf.py --workers 125,250,500,1000,2000,4000 --cps 1 --rounds 1 | sed "s/^{/{\"variant\": \"$v\", \"rep\": $r, /" >> $F/ab.jsonl
  done
done
cp abtest/new.so $L
timeout 600 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "interleaved or randomized" 2>&1 | tail -3 > $F/pytest.log
