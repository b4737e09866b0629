# Scratch driver for one gpurun call (edited per experiment).
set -x
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/final/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
for i in 1 2 3; do timeout 600 python bench.py 2>>gpurun_out/final/bench.err >> gpurun_out/final/bench.jsonl; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 20 --warmup 3 > gpurun_out/final/bench_under_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -f -o /tmp/prof_all python tools/profile_all.py > gpurun_out/final/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof_all.ncu-rep -o gpurun_out/final/ncu_full_all_kernels.json >> gpurun_out/final/ncu_full.log 2>&1
