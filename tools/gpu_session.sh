# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/final5
mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $F/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1
oracle/_ref/ref_tests_on_b200 2>&1 | tail -2 > $F/ref_tests.log
timeout 600 python bench.py 2>$F/bench.err > $F/bench.json
timeout 600 python bench.py --impl reference > $F/bench_reference.json 2>> $F/bench.err
