F=gpurun_out/s38; mkdir -p $F
BCN_DEINT_NARROW_HUGE_MIN_U32=32 BCN_FUZZ_CASES_DEINT=200 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest.log 2>&1; echo "rc=$?" >> $F/pytest.log
W=33,48,63,65,72,85,100,116,127
for rep in 1 2; do for m in 100000 32; do
for l in 30 28; do BCN_DEINT_NARROW_HUGE_MIN_U32=$m BCN_DEINT_LOG2N=$l timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"m\": $m, \"log2n\": $l, /" >> $F/d.jsonl 2>>$F/err.txt; done
done; done
