# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/final4
mkdir -p $F
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $F/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $F/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1
oracle/_ref/ref_tests_on_b200 2>&1 | tail -2 > $F/ref_tests.log
timeout 600 python bench.py --impl reference > $F/bench_reference.json 2> $F/bench_reference.err
for i in 1 2 3; do timeout 600 python bench.py 2>>$F/bench.err >> $F/bench.jsonl; done
for tool in memcheck racecheck; do
  echo "## $tool" >> $F/san.txt
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool python tools/sanitize.py 2>&1 | grep -v "^========= *$" | tail -4 >> $F/san.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench.csv python bench.py --steps 20 --warmup 3 > $F/bench_under_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -f -o /tmp/prof_all python tools/profile_all.py > $F/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof_all.ncu-rep -o $F/ncu_full_all_kernels.json >> $F/ncu_full.log 2>&1
