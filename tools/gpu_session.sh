# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 tools/c/device_api_perf_old | sed 's/^{/{"header": "int128-mod", /' > gpurun_out/device_api.jsonl 2>>gpurun_out/err.log
timeout 300 tools/c/device_api_perf | sed 's/^{/{"header": "barrett", /' >> gpurun_out/device_api.jsonl 2>>gpurun_out/err.log
