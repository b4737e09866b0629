set -x
F=gpurun_out/s11
mkdir -p $F
nvidia-smi --query-gpu=name,serial,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $F/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo "smoke rc=$?" >> $F/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > $F/pytest.log 2>&1; echo "pytest rc=$?" >> $F/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $F/bench_default.json 2> $F/bench_default.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $F/bench_reference_arm.json 2> $F/bench_reference_arm.err
BCN_PACE_CALIBRATE=0 timeout 1200 compute-sanitizer --tool synccheck python tools/sanitize.py > $F/sanitize_synccheck.txt 2>&1; echo "rc=$?" >> $F/sanitize_synccheck.txt
ls -la $F
