F=gpurun_out/s19; mkdir -p $F
W=65,85,100,127,129,200,1000,5003,100003,1000000
for rep in 1 2; do
BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"base\", /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_U32_NARROW_MAX=64 BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"u32wide\", /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_U32_NARROW_MAX=64 BCN_DEINT_ALIGN=2 BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"u32wide_halo\", /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_HALO_LINE=1 BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"line\", /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_U32_NARROW_MAX=64 BCN_DEINT_ALIGN=2 BCN_DEINT_HALO_LINE=1 BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"u32wide_halo_line\", /" >> $F/d.jsonl 2>>$F/err.txt
done
BCN_DEINT_HALO_LINE=1 BCN_FUZZ_CASES_DEINT=300 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest_line.log 2>&1; echo "rc=$?" >> $F/pytest_line.log
BCN_DEINT_U32_NARROW_MAX=64 BCN_DEINT_ALIGN=2 BCN_FUZZ_CASES_DEINT=300 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave" > $F/pytest_wide2.log 2>&1; echo "rc=$?" >> $F/pytest_wide2.log
tail -3 $F/err.txt
