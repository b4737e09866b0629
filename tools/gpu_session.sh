# Scratch driver for one gpurun call (edited per experiment).
set -x
oracle/_ref/ref_tests_on_b200 > gpurun_out/ref_tests.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
