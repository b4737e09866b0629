F=gpurun_out/s16i; mkdir -p $F
BCN_FUZZ_CASES_DEINT=600 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave or interleaved" > $F/pytest_deint.log 2>&1; echo "rc=$?" >> $F/pytest_deint.log
for m in 0 1; do
BCN_DEINT_ALIGN=$m timeout 600 python tools/deint_align.py | sed "s/^{/{\"align\": $m, /" >> $F/deint_align.jsonl 2>> $F/err.txt
done
W=1,2,7,16,31,33,64,85,86,100,128,129,200,1000,5003,100003,1000000
for m in 0 1; do
BCN_DEINT_ALIGN=$m BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"align\": $m, \"log2n\": 30, /" >> $F/deint_final.jsonl 2>>$F/err.txt
BCN_DEINT_ALIGN=$m BCN_DEINT_LOG2N=28 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"align\": $m, \"log2n\": 28, /" >> $F/deint_final.jsonl 2>>$F/err.txt
done
tail -3 $F/err.txt
