# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/cli
mkdir -p $F
oracle/_ref/ref_tests_on_b200 > $F/ref_tests.log 2>&1
timeout 900 python -m pytest tests/test_dropin.py -m gpu -q 2>&1 | tail -5 > $F/pytest.log
(time tests/cpp/build/bcnrand gen --n 100000000 --format raw-f64 --out /tmp/big.f64) > $F/gen_time.log 2>&1
(time tests/cpp/build/bcnrand gen --n 20000000 --format text --out /tmp/big.txt) >> $F/gen_time.log 2>&1
ls -la /tmp/big.f64 /tmp/big.txt >> $F/gen_time.log
tests/cpp/build/bcnrand bench --repeats 3 > $F/bench.txt 2>&1; tests/cpp/build/bcnrand bench --n 1073741824 --repeats 5 --csv >> $F/bench.txt 2>&1
tests/cpp/build/bcnrand selftest > $F/selftest.txt 2>&1
