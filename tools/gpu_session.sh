# Scratch driver for one gpurun call (edited per experiment).
set -x
timeout 600 python tools/inter_perf.py --workers 7,125,250,500,1000,1024,1536,2000 --cps 1 --rounds 2 > gpurun_out/inter.jsonl 2>>gpurun_out/err.log
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:k_fill_paced --csv --log-file gpurun_out/inter_launches.csv python tools/inter_perf.py --workers 7,1000,1024 --cps 1 --rounds 1 > /dev/null 2>&1
