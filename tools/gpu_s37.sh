F=gpurun_out/s37; mkdir -p $F
BCN_FUZZ_CASES_DEINT=400 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest.log 2>&1; echo "rc=$?" >> $F/pytest.log
W=132,200,1000,1024,4096,100000,1000000
for rep in 1 2; do for m in 0 1; do
for l in 30 28; do BCN_DEINT_VEC_LOADS=$m BCN_DEINT_LOG2N=$l timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"m\": $m, \"log2n\": $l, /" >> $F/d.jsonl 2>>$F/err.txt; done
done; done
for m in 0 1; do BCN_DEINT_VEC_LOADS=$m timeout 600 python tools/deint_align.py | sed "s/^{/{\"m\": $m, /" >> $F/align.jsonl 2>> $F/err.txt; done
