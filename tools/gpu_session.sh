# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/pace
mkdir -p $F
for r in 1 2; do
  for p in 7200 6800 7000 7400 6600; do
    timeout 600 python bench.py --pace $p --no-cpu 2>>$F/err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(json.dumps({'pace': $p, 'rep': $r, 'value': d['value'], 'gbs': d['roofline']['achieved'], 'noise': d['roofline'].get('noise_writer_gbs'), 'clk_mean': d['clocks'].get('sm_mhz_mean'), 'power': d['clocks'].get('power_w_median')}))" >> $F/pace.jsonl
  done
done
