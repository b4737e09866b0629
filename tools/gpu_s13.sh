set -x
F=gpurun_out/s13b
mkdir -p $F
timeout 600 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave or interleaved" -x > $F/pytest_deint.log 2>&1; echo "rc=$?" >> $F/pytest_deint.log
W=1024,4096,65536,1048576,1000,1000000
for rep in 1 2; do
  BCN_DEINT_LOG2N=30 BCN_DEINT_TMA=1 timeout 300 python tools/deint_perf.py $W >> $F/deint_ab.jsonl 2>>$F/deint.err
  BCN_DEINT_LOG2N=30 BCN_DEINT_TMA=0 timeout 300 python tools/deint_perf.py $W >> $F/deint_ab.jsonl 2>>$F/deint.err
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:transpose_tma -c 1 -o /tmp/tma_w4096_i4 python tools/deint_one.py --w 4096 --isz 4 --log2n 30 > $F/ncu.log 2>&1
ncu -i /tmp/tma_w4096_i4.ncu-rep --page details --csv > $F/details_tma_w4096_i4.csv 2>/dev/null
ncu -i /tmp/tma_w4096_i4.ncu-rep --page raw --csv > $F/raw_tma_w4096_i4.csv 2>/dev/null
ls -la $F
