# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 --sweep gpurun_out/sweep.jsonl > gpurun_out/bench_sweep.json 2>>gpurun_out/err.log
