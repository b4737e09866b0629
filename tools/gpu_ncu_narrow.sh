F=gpurun_out/s30; mkdir -p $F
for w in 64 65 100; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transpose_narrow -c 1 -o /tmp/n$w python tools/deint_one.py --w $w --isz 4 --log2n 30 > $F/ncu$w.log 2>&1
ncu -i /tmp/n$w.ncu-rep --page details --csv > $F/details_$w.csv 2>/dev/null
ncu -i /tmp/n$w.ncu-rep --page raw --csv > $F/raw_$w.csv 2>/dev/null
ncu -i /tmp/n$w.ncu-rep --page source --csv --print-source sass > $F/src_$w.csv 2>/dev/null
done
