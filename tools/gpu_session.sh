# Scratch driver for one gpurun call (edited per experiment).
set -x
L=paper_1206_1187_b200/libbcnrand_b200.so
cp $L /tmp/lib_current.so
for rep in 1 2; do for v in bar common; do
  cp abtest/lib_$v.so $L; touch $L
  timeout 120 python tools/timeline.py --pace 7200 --cps 1 --launches 400 --tag $v >> gpurun_out/ab_barrier.jsonl 2>>gpurun_out/err.log
  timeout 300 python tools/tune.py --fmts f64 --engines FP64 --pace 7200 --cps 1 --rounds 3 | sed "s/^{/{\"tag\": \"$v\", /" >> gpurun_out/ab_barrier_tune.jsonl 2>>gpurun_out/err.log
done; done
cp /tmp/lib_current.so $L; touch $L
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_synccheck.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
