# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/narrow2
mkdir -p $F
timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "deinterleave or interleaved or randomized" 2>&1 | tail -3 > $F/pytest.log
timeout 300 python tools/deint_perf.py > $F/final.jsonl
timeout 300 python tools/deint_perf.py 80,86,90,100,120 >> $F/final.jsonl
