# Scratch driver for one gpurun call (edited per experiment).
set -x
mkdir -p gpurun_out/deint
timeout 600 python -m pytest tests/test_gpu_fill.py -m gpu -q -k "deinterleave or interleaved" 2>&1 | tail -3 > gpurun_out/deint/pytest2.log
timeout 300 python tools/deint_perf.py > gpurun_out/deint/final2.jsonl
timeout 300 python tools/deint_perf.py 65,80,100,5000,20000,1000003 >> gpurun_out/deint/final2.jsonl
