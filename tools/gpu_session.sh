# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s2
mkdir -p $F
for rep in 1 2; do
  for fl in 0 2 1 3; do
    BCN_PACE_FLAGS=$fl timeout 300 python tools/pace_modes.py --tag rep$rep >> $F/pace_modes.jsonl 2>>$F/err.log
  done
done
