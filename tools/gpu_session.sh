# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/fuzz
mkdir -p $F
BCN_FUZZ_CASES=5000 BCN_FUZZ_CASES_DEINT=1500 timeout 2400 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "randomized" 2>&1 | tail -3 > $F/fuzz.log
