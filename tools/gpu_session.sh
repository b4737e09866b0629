# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 300 python bench.py > gpurun_out/bench_default.json 2>>gpurun_out/err.log
timeout 300 python bench.py --impl reference > gpurun_out/bench_reference_arm.json 2>>gpurun_out/err.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -o /tmp/prof_all python tools/profile_all.py > gpurun_out/prof_all.log 2>&1
python tools/ncu_summary.py /tmp/prof_all.ncu-rep -o gpurun_out/ncu_full_all_kernels.json >> gpurun_out/prof_all.log 2>&1
