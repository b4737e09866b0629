F=gpurun_out/s25; mkdir -p $F
BCN_FUZZ_CASES_DEINT=600 timeout 900 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "deinterleave or interleaved" > $F/pytest_deint.log 2>&1; echo "rc=$?" >> $F/pytest_deint.log
W=1,2,7,16,31,33,64,65,85,86,100,120,127,128,129,200,1000,5003,100003,1000000
BCN_DEINT_LOG2N=30 timeout 600 python tools/deint_perf.py $W > $F/deinterleave_final_2e30.jsonl 2>> $F/deint.err
BCN_DEINT_LOG2N=28 timeout 600 python tools/deint_perf.py $W > $F/deinterleave_final_2e28.jsonl 2>> $F/deint.err
