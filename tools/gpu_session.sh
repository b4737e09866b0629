# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "seed" 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:k_seed --csv --log-file gpurun_out/seed_launches.csv python tools/secondary_perf.py > /dev/null 2>&1
