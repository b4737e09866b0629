# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s1
mkdir -p $F
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $F/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $F/pytest.log 2>&1
echo "pytest rc=$?" >> $F/pytest.log
for fmt in f64 u64; do
  timeout 300 python tools/ab_lib.py --libs abtest/r01.so,paper_1206_1187_b200/libbcnrand_b200.so --fmt $fmt --pace 7200 --tag mbar_vs_bar >> $F/ab.jsonl 2>>$F/ab.err
  timeout 300 python tools/ab_lib.py --libs abtest/r01.so,paper_1206_1187_b200/libbcnrand_b200.so --fmt $fmt --tag default >> $F/ab.jsonl 2>>$F/ab.err
done
timeout 600 python bench.py --steps 20 --warmup 5 > $F/bench.json 2> $F/bench.err
BCN_PACE_CALIBRATE=0 timeout 900 compute-sanitizer --tool synccheck python tools/sanitize.py > $F/synccheck.txt 2>&1
echo "synccheck rc=$?" >> $F/synccheck.txt
