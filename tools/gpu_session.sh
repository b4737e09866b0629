# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python tools/hostfill_perf.py >> gpurun_out/hostfill.jsonl 2>>gpurun_out/err.log
