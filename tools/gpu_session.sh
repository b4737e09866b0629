# Final evidence pass on the round-2 code (one gpurun call); outputs under gpurun_out/final.
set -x
F=gpurun_out/final3
mkdir -p $F
nvidia-smi --query-gpu=name,serial,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $F/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo "smoke rc=$?" >> $F/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > $F/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $F/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $F/bench_default.json 2> $F/bench_default.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $F/bench_reference_arm.json 2> $F/bench_reference_arm.err
PACE=$(python -c "import json;print(json.load(open('$F/bench_default.json'))['launch']['write_pacing_gbs'])")
for v in "--fmt u64" "--fmt f32" "--engine barrett" "--engine montgomery" "--engine staged" "--engine bulk" "--engine mixed" "--engine hybrid" "--fmt f32 --engine hybrid"; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-c5 $v >> $F/bench_variants.jsonl 2>> $F/bench_variants.err
done
timeout 900 python bench.py --workload c5 --steps 5 --warmup 2 --no-cpu --no-e2e > $F/bench_c5.json 2>> $F/bench_c5.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-c5 --sustain-s 0 --sweep $F/sweep_c3.jsonl > /dev/null 2>> $F/sweep.err
W=1,2,7,16,31,33,64,65,85,86,100,128,129,200,1000,5003,100003,1000000
BCN_DEINT_LOG2N=30 timeout 600 python tools/deint_perf.py $W > $F/deinterleave_final_2e30.jsonl 2>> $F/deint.err
BCN_DEINT_LOG2N=28 timeout 600 python tools/deint_perf.py $W > $F/deinterleave_final_2e28.jsonl 2>> $F/deint.err
for W in 7 64 125 250 1001 5003 20000 100003; do
  timeout 300 python tools/ab_lib.py --libs paper_1206_1187_b200/libbcnrand_b200.so --fmt f64 --interleaved --workers $W --rounds 4 --tag interleaved_final >> $F/interleaved_final.jsonl 2>>$F/inter.err
done
BCN_PACE_CALIBRATE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-c5 --sustain-s 0 --pace $PACE > $F/launches_bench.log 2>&1
BCN_PACE_CALIBRATE=0 timeout 1800 ncu --set full --clock-control none --import-source on -o /tmp/prof_all python tools/profile_all.py --pace $PACE > $F/prof_all.log 2>&1
python tools/ncu_summary.py /tmp/prof_all.ncu-rep -o $F/ncu_full_all_kernels.json >> $F/prof_all.log 2>&1
python tools/ncu_summary.py --launches $F/launches_bench.csv -o $F/launches_bench.json >> $F/prof_all.log 2>&1
for tool in memcheck racecheck synccheck; do
  BCN_PACE_CALIBRATE=0 timeout 1200 compute-sanitizer --tool $tool python tools/sanitize.py > $F/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> $F/sanitize_$tool.txt
done
cuobjdump -sass paper_1206_1187_b200/libbcnrand_b200.so | grep -E "Function|UTMALDG|UTMASTG|STG.E.ENL2.256|STG.E.128|UBLKCP" | sort | uniq -c | sort -rn | head -60 > $F/sass_inventory.txt
ls -la $F
