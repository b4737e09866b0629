# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_digest --csv --log-file gpurun_out/digest_launches.csv python tools/profile_all.py > /dev/null 2>&1
