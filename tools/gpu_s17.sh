F=gpurun_out/s17b; mkdir -p $F
BCN_FUZZ_CASES_DEINT=600 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave or interleaved" > $F/pytest_deint.log 2>&1; echo "rc=$?" >> $F/pytest_deint.log
W=8,9,16,31,33,48,63,64,65,85,100,127,128
for rep in 1 2; do
for m in 0 1; do
BCN_DEINT_NARROW_HALO=$m BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"nhalo\": $m, \"log2n\": 30, /" >> $F/deint_narrow.jsonl 2>>$F/err.txt
BCN_DEINT_NARROW_HALO=$m BCN_DEINT_LOG2N=28 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"nhalo\": $m, \"log2n\": 28, /" >> $F/deint_narrow.jsonl 2>>$F/err.txt
done; done
tail -3 $F/err.txt
