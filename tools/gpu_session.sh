# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s5
mkdir -p $F
M="--set full --clock-control none --import-source on"
for cfg in "0 4 1000000" "1 4 1000000" "0 4 200" "1 4 200" "0 8 86" "1 8 86" "0 8 1000000" "0 4 100"; do
  set -- $cfg
  R=/tmp/deint_b$1_i$2_w$3
  BCN_DEINT_BULK=$1 timeout 600 ncu $M -k regex:"transpose|deint" -s 3 -c 1 -o $R python tools/deint_one.py --isz $2 --w $3 > $F/ncu_b$1_i$2_w$3.log 2>&1
  ncu -i $R.ncu-rep --page raw --csv > $F/raw_b$1_i$2_w$3.csv 2>&1
  ncu -i $R.ncu-rep --page details --csv > $F/details_b$1_i$2_w$3.csv 2>&1
done
ls -la $F
