# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 1 python tools/sanitize.py > gpurun_out/sanitize_initcheck.log 2>&1
