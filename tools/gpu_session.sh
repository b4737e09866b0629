# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k quality 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/quality_launches.csv python tools/quality_perf.py > gpurun_out/quality_perf.log 2>&1
