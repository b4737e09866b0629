# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k quality 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_monobit --csv --log-file gpurun_out/mono_launches.csv python tools/quality_perf.py > gpurun_out/qp.log 2>&1
