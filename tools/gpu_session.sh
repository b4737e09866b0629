# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s9
mkdir -p $F
for cps in 1 2 3; do
  for pace in 6800 7200; do
    timeout 300 python tools/ab_lib.py --libs paper_1206_1187_b200/libbcnrand_b200.so,abtest/f32h2.so --fmt f32 --pace $pace --cps $cps --mask 7 --rounds 6 --tag f32h2 >> $F/f32h2.jsonl 2>>$F/err.log
  done
done
timeout 300 python tools/ab_lib.py --libs paper_1206_1187_b200/libbcnrand_b200.so --fmt f32 --pace 0 --rounds 6 --tag f32unpaced >> $F/f32h2.jsonl 2>>$F/err.log
