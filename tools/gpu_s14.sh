F=gpurun_out/s14; mkdir -p $F
for args in "100003 129 4" "100003 1000 8" "1000000 1000 4"; do
  timeout 300 compute-sanitizer --show-backtrace device python tools/deint_dbg.py $args > $F/san_$(echo $args | tr ' ' _).txt 2>&1
done
cuobjdump -sass -fun regex:k_transpose_tma paper_1206_1187_b200/libbcnrand_b200.so > $F/sass_tma.txt 2>&1
ls -la $F
