F=gpurun_out/s18; mkdir -p $F
for m in 0 1; do
BCN_DEINT_NARROW_HALO=$m timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transpose_narrow -c 1 -o /tmp/nh$m python tools/deint_one.py --w 100 --isz 4 --log2n 28 > $F/ncu$m.log 2>&1
ncu -i /tmp/nh$m.ncu-rep --page details --csv > $F/details_nh$m.csv 2>/dev/null
ncu -i /tmp/nh$m.ncu-rep --page raw --csv > $F/raw_nh$m.csv 2>/dev/null
ncu -i /tmp/nh$m.ncu-rep --page source --csv --print-source sass > $F/src_nh$m.csv 2>/dev/null
done
