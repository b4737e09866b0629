# Exploration call: hybrid-engine f32 A/B and source-level ncu of the wide deinterleave.
set -x
F=gpurun_out/s12
mkdir -p $F
L=paper_1206_1187_b200/libbcnrand_b200.so
for rep in 1 2; do
  timeout 300 python tools/ab_lib.py --libs $L --fmt f32 --engine 3 --tag fp64_unpaced >> $F/hybrid.jsonl 2>>$F/hybrid.err
  for kf in 7 6 5; do
    BCN_HYBRID_KF=$kf timeout 300 python tools/ab_lib.py --libs $L --fmt f32 --engine 7 --tag hybrid_kf$kf >> $F/hybrid.jsonl 2>>$F/hybrid.err
  done
  for kf in 7 6; do
    BCN_HYBRID_KF=$kf timeout 300 python tools/ab_lib.py --libs $L --fmt f32 --engine 7 --pace 6800 --mask 7 --cps 2 --tag hybrid_paced_kf$kf >> $F/hybrid.jsonl 2>>$F/hybrid.err
  done
  timeout 300 python tools/ab_lib.py --libs $L --fmt f32 --engine 3 --pace 6800 --mask 7 --cps 2 --tag fp64_paced >> $F/hybrid.jsonl 2>>$F/hybrid.err
  BCN_HYBRID_KF=3 timeout 300 python tools/ab_lib.py --libs $L --fmt f64 --engine 7 --tag hybrid_f64_kf3 >> $F/hybrid.jsonl 2>>$F/hybrid.err
done
python - > $F/deint_2e30.jsonl 2>$F/deint.err <<'PY'
import json, statistics, torch, paper_1206_1187_b200 as B
dev = torch.device("cuda:0"); st = torch.cuda.current_stream(dev)
for log2n in (28, 30):
    n = 1 << log2n
    for dt, isz in ((torch.float64, 8), (torch.float32, 4)):
        buf = torch.empty(n, dtype=dt, device=dev)
        for w in (7, 64, 100, 1000, 5003, 100003, 1000000):
            plan = B.par.make_plan(n, w, B.Layout.Interleaved)
            B.par.deinterleave(buf, plan)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
            ev[0].record(st)
            for i in range(10):
                B.par.deinterleave(buf, plan); ev[i + 1].record(st)
            torch.cuda.synchronize()
            ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(10))
            print(json.dumps({"log2n": log2n, "itemsize": isz, "workers": w, "ms": ms, "gbs_rw": 2 * n * isz / ms / 1e6}), flush=True)
        del buf
PY
for w in 1000000 1000; do
  for isz in 8 4; do
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:transpose -c 1 -o /tmp/deint_w${w}_i${isz} python tools/deint_one.py --w $w --isz $isz --log2n 30 > $F/ncu_w${w}_i${isz}.log 2>&1
    ncu -i /tmp/deint_w${w}_i${isz}.ncu-rep --page source --csv --print-source sass > $F/src_w${w}_i${isz}.csv 2>/dev/null
    ncu -i /tmp/deint_w${w}_i${isz}.ncu-rep --page raw --csv > $F/raw_w${w}_i${isz}.csv 2>/dev/null
    ncu -i /tmp/deint_w${w}_i${isz}.ncu-rep --page details --csv > $F/details_w${w}_i${isz}.csv 2>/dev/null
  done
done
ls -la $F
