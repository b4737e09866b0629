F=gpurun_out/s36; mkdir -p $F
BCN_DEINT_WIDE=7 BCN_DEINT_WIDE_THREADS=512 BCN_FUZZ_CASES_DEINT=200 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest.log 2>&1; echo "rc=$?" >> $F/pytest.log
W=129,200,1000,5003,100003,1000000
for rep in 1 2; do
for l in 30 28; do BCN_DEINT_LOG2N=$l timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"base\", \"log2n\": $l, /" >> $F/d.jsonl 2>>$F/err.txt; done
for l in 30 28; do BCN_DEINT_WIDE=7 BCN_DEINT_WIDE_THREADS=512 BCN_DEINT_LOG2N=$l timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"t256x256\", \"log2n\": $l, /" >> $F/d.jsonl 2>>$F/err.txt; done
done
