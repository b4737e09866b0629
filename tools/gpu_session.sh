# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s4
mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $F/pytest.log 2>&1; echo "pytest rc=$?" >> $F/pytest.log
W=7,64,85,86,100,128,129,200,1000,5003,100003,1000000
for v in 0 1 2 3; do
  BCN_DEINT_BULK=$v timeout 600 python tools/deint_perf.py $W | sed "s/^{/{\"bulk\": $v, /" >> $F/deint.jsonl 2>>$F/deint.err
done
timeout 600 python bench.py --steps 20 --warmup 5 > $F/bench.json 2> $F/bench.err
