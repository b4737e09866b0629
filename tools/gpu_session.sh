# Scratch driver for one gpurun call (edited per experiment).
set -x
for p in 7200 6400 6800 7200 6000; do
  timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 5 --pace $p | sed "s/^{/{\"pace_arg\": $p, /" >> gpurun_out/c5_pace.jsonl 2>>gpurun_out/err.log
  sleep 20
done
