F=gpurun_out/s20; mkdir -p $F
W=96,100,101,104,108,112,116,120,124,127,128
for rep in 1 2; do
BCN_DEINT_U32_NARROW_MAX=128 BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"narrow\", /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_U32_NARROW_MAX=64 BCN_DEINT_LOG2N=30 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"wide\", /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_U32_NARROW_MAX=128 BCN_DEINT_LOG2N=28 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"narrow28\", /" >> $F/d.jsonl 2>>$F/err.txt
BCN_DEINT_U32_NARROW_MAX=64 BCN_DEINT_LOG2N=28 timeout 300 python tools/deint_perf.py $W | sed "s/^{/{\"v\": \"wide28\", /" >> $F/d.jsonl 2>>$F/err.txt
done
