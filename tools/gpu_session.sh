set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for s in 1 0 1 0; do BCN_PACE_STAGGER=$s timeout 300 python bench.py --no-cpu > gpurun_out/bench_stagger$s.$RANDOM.json 2>gpurun_out/bench_err.log; done
for s in 1 0; do BCN_PACE_STAGGER=$s timeout 600 python tools/tune.py --fmts f64 --engines FP64 --pace 6800,7000,7200,7400,7600 --cps 2 --rounds 4 > gpurun_out/tune_stagger$s.jsonl 2>&1; done
timeout 300 python bench.py > gpurun_out/bench_default.json 2>>gpurun_out/bench_err.log
