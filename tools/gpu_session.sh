# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s6
mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $F/pytest.log 2>&1; echo "pytest rc=$?" >> $F/pytest.log
for W in 7 64 125 250 1001 5003 100003; do
  timeout 300 python tools/ab_lib.py --libs abtest/r01.so,paper_1206_1187_b200/libbcnrand_b200.so --fmt f64 --pace 7200 --interleaved --workers $W --rounds 8 --tag inter >> $F/inter.jsonl 2>>$F/inter.err
done
W=7,64,86,100,128,129,200,1000,5003,100003,1000000
for v in 0 1 2 3; do
  BCN_DEINT_BULK=$v timeout 600 python tools/deint_perf.py $W | sed "s/^{/{\"bulk\": $v, /" >> $F/deint.jsonl 2>>$F/deint.err
done
