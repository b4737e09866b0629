F=gpurun_out/s24; mkdir -p $F
BCN_DEINT_NARROW_THREADS=512 BCN_DEINT_WIDE_THREADS=512 BCN_DEINT_MINB=2 BCN_FUZZ_CASES_DEINT=300 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest512.log 2>&1; echo "rc=$?" >> $F/pytest512.log
W=2,7,16,31,48,64,65,85,100,116,120,127,129,200,1000,5003,100003,1000000
for rep in 1 2; do
BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"base\", \"log2n\": 30, /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_NARROW_THREADS=512 BCN_DEINT_WIDE_THREADS=512 BCN_DEINT_MINB=2 BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"nt512m2\", \"log2n\": 30, /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_LOG2N=28 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"base\", \"log2n\": 28, /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_NARROW_THREADS=512 BCN_DEINT_WIDE_THREADS=512 BCN_DEINT_MINB=2 BCN_DEINT_LOG2N=28 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"nt512m2\", \"log2n\": 28, /" >> $F/d.jsonl 2>>$F/err.txt
done
