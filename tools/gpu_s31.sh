F=gpurun_out/s31; mkdir -p $F
BCN_FUZZ_CASES_DEINT=400 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest.log 2>&1; echo "rc=$?" >> $F/pytest.log
W=1,2,7,9,16,31,33,48,63,64,65,85,100,116
for l in 30 28; do BCN_DEINT_LOG2N=$l timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"log2n\": $l, /" >> $F/d.jsonl 2>>$F/err.txt; done
timeout 600 ncu --set full --clock-control none -k regex:k_transpose_narrow -c 1 -o /tmp/n65 python tools/deint_one.py --w 65 --isz 4 --log2n 30 > $F/ncu.log 2>&1
ncu -i /tmp/n65.ncu-rep --page raw --csv > $F/raw_65.csv 2>/dev/null
