F=gpurun_out/s34; mkdir -p $F
BCN_DEINT_NARROW_BIG_MIN_U32=8 BCN_DEINT_NARROW_BIG_MIN_U64=8 BCN_FUZZ_CASES_DEINT=300 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest.log 2>&1; echo "rc=$?" >> $F/pytest.log
W=9,16,31,33,48,63,64,65,85,100,116
for rep in 1 2; do for m in 1000 8; do
for l in 30 28; do BCN_DEINT_NARROW_BIG_MIN_U32=$m BCN_DEINT_NARROW_BIG_MIN_U64=$m BCN_DEINT_LOG2N=$l timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"m\": $m, \"log2n\": $l, /" >> $F/d.jsonl 2>>$F/err.txt; done
done; done
