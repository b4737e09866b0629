F=gpurun_out/s35; mkdir -p $F
BCN_FUZZ_CASES_DEINT=400 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave or interleaved" > $F/pytest.log 2>&1; echo "rc=$?" >> $F/pytest.log
W=100,116,117,120,124,127,128,129
for rep in 1 2; do for m in 116 128; do
for l in 30 28; do BCN_DEINT_U32_NARROW_MAX=$m BCN_DEINT_LOG2N=$l timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"nmax\": $m, \"log2n\": $l, /" >> $F/d.jsonl 2>>$F/err.txt; done
done; done
