# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/s8
mkdir -p $F
W=129,200,1000,5003,100003,1000000
for v in 0 1 2 3 4 5 6; do
  BCN_DEINT_WIDE=$v timeout 600 python tools/deint_perf.py $W | sed "s/^{/{\"wide\": $v, /" >> $F/deint.jsonl 2>>$F/deint.err
done
for cps in 2 3 4; do
  python - >> $F/f32_paced.jsonl 2>>$F/f32.err <<PY
import json, statistics, torch, paper_1206_1187_b200 as B
n = 1 << 30
buf = torch.empty(n, dtype=torch.float32, device="cuda:0")
plan = B.par.make_plan(n, 1)
s = torch.cuda.current_stream()
for pace in (0, 6400, 6800, 7200):
    B.device.set_write_pacing(pace if pace else -1, $cps, 7 if pace else 3)
    f = lambda: B.par.fill_float(buf, plan, B.kMinSeedIndex, stream=s)
    for _ in range(3): f()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
    ev[0].record(s)
    for i in range(20):
        f(); ev[i + 1].record(s)
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(20)]
    print(json.dumps({"fmt": "f32", "cps": $cps, "pace": pace, "median_gbs": 4 * n / statistics.median(ms) / 1e6, "best_gbs": 4 * n / min(ms) / 1e6}))
PY
done
