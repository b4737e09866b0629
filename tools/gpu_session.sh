# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 tools/c/latency > gpurun_out/latency.jsonl 2>>gpurun_out/err.log
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_memcheck.log 2>&1
timeout 300 python bench.py --no-cpu > gpurun_out/bench.json 2>>gpurun_out/err.log
