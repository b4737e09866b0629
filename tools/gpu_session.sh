# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/pitch4
mkdir -p $F
timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "deinterleave or interleaved or randomized" 2>&1 | tail -3 > $F/pytest.log
timeout 300 python tools/deint_perf.py 3,4,5,6,7,8,9,16 | grep '"itemsize": 4' > $F/final.jsonl
