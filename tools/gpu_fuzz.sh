# Extended randomized parity (fill + deinterleave fuzz scaled up), round 2 code.
F=gpurun_out/fuzz; mkdir -p $F
BCN_FUZZ_CASES=5000 BCN_FUZZ_CASES_DEINT=3000 timeout 3000 python -m pytest tests/test_gpu_fill.py -m gpu -q -p no:cacheprovider -k "randomized" --durations=5 > $F/fuzz_extended.txt 2>&1; echo "rc=$?" >> $F/fuzz_extended.txt
