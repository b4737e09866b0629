# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s7
mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $F/pytest.log 2>&1; echo "pytest rc=$?" >> $F/pytest.log
for W in 7 125 250 1001 5003 20000 100003; do
  timeout 300 python tools/ab_lib.py --libs abtest/r01.so,paper_1206_1187_b200/libbcnrand_b200.so --fmt f64 --pace 7200 --interleaved --workers $W --rounds 8 --tag inter >> $F/inter.jsonl 2>>$F/inter.err
done
timeout 600 python bench.py --steps 20 --warmup 5 > $F/bench.json 2> $F/bench.err
