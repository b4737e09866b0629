# Scratch driver for one gpurun call (edited per experiment).
set -x
nvidia-smi --query-gpu=name,serial,temperature.gpu,power.draw,clocks.sm --format=csv > gpurun_out/box.txt
for i in 1 2 3; do timeout 300 python bench.py --no-cpu >> gpurun_out/bench_repeat.jsonl 2>>gpurun_out/err.log; sleep 10; done
timeout 900 python -m pytest tests -m gpu -x -q -k "cli" 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
