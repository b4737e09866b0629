# Scratch driver for one gpurun call (edited per experiment).
set -x
mkdir -p gpurun_out/deint
timeout 600 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "randomized_deinterleave" 2>&1 | tail -5 > gpurun_out/deint/fuzz.log
