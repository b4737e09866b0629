# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/variants
mkdir -p $F
for a in "--fmt u64" "--fmt f32" "--engine barrett" "--engine montgomery" "--engine staged" "--engine bulk"; do
  timeout 600 python bench.py $a --no-cpu >> $F/bench_variants.jsonl 2>> $F/err.log || echo "FAILED $a" >> $F/err.log
done
