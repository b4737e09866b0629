# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/inter
mkdir -p $F
for r in 1 2; do
  for v in 1 0; do
    BCN_INTER_FIXED=$v timeout 300 python tools/inter_perf.py --workers 7,64,125,250,1000,1024,1536,2000 --cps 1 --rounds 1 | sed "s/^{/{\"fixed\": $v, \"rep\": $r, /" >> $F/fixed_vs_two.jsonl
  done
done
