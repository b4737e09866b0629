F=gpurun_out/s23; mkdir -p $F
BCN_DEINT_WIDE_THREADS=512 BCN_FUZZ_CASES_DEINT=300 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest512.log 2>&1; echo "rc=$?" >> $F/pytest512.log
timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest.log 2>&1; echo "rc=$?" >> $F/pytest.log
W=2,16,31,33,48,64,65,85,86,100,120,127,129,200,1000,5003,100003,1000000
for rep in 1 2; do for nt in 256 512; do
BCN_DEINT_WIDE_THREADS=$nt BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"nt\": $nt, \"log2n\": 30, /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_WIDE_THREADS=$nt BCN_DEINT_LOG2N=28 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"nt\": $nt, \"log2n\": 28, /" >> $F/d.jsonl 2>>$F/err.txt
done; done
