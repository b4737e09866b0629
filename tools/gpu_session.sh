# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "deinterleave or invariance or ragged" 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python tools/deint_perf.py >> gpurun_out/deint.jsonl 2>>gpurun_out/err.log
