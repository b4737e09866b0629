F=gpurun_out/s26; mkdir -p $F
for w in 1000 129; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transpose -c 1 -o /tmp/u32_$w python tools/deint_one.py --w $w --isz 4 --log2n 30 > $F/ncu_$w.log 2>&1
ncu -i /tmp/u32_$w.ncu-rep --page details --csv > $F/details_$w.csv 2>/dev/null
ncu -i /tmp/u32_$w.ncu-rep --page raw --csv > $F/raw_$w.csv 2>/dev/null
ncu -i /tmp/u32_$w.ncu-rep --page source --csv --print-source sass > $F/src_$w.csv 2>/dev/null
done
