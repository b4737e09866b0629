#!/usr/bin/env python
"""Render the committed `ncu --set full` summary as a per-kernel markdown table
(evidence view): for the largest captured launch of every kernel, its time,
DRAM write rate and share of peak, issue activity and pipe utilisation — the
FP64 pipe for the FP64 engine, the FMA pipe (IMAD: the integer multiplies of
the Barrett / Montgomery / modified-Barrett engines) and ALU for the integer
ones, LSU for the stores.

    python tools/ncu_table.py profiles/r01/ncu_full_all_kernels.json > profiles/r01/ncu_table.md
"""
from __future__ import annotations

import json
import sys


def main() -> None:
    rows = json.load(open(sys.argv[1]))
    best: dict[str, dict] = {}
    for r in rows:
        k = r["kernel"].strip()
        if k not in best or r["gpu__time_duration.sum"] > best[k]["gpu__time_duration.sum"]:
            best[k] = r
    print("| kernel (largest captured launch) | ms | DRAM write GB/s | DRAM % peak | issue % | FP64 pipe % | FMA/IMAD pipe % | ALU pipe % | LSU % | regs | grid x block |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for k, r in sorted(best.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        ms = r["gpu__time_duration.sum"]  # ncu_summary stores msecond
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        wbytes = r["dram__bytes_write.sum"] * scale[r.get("dram__bytes_write.sum.unit", "byte")]
        wr = wbytes / (ms * 1e-3) / 1e9
        f = lambda key: r.get(key, float("nan"))  # noqa: E731
        print(f"| `{k}` | {ms:.3f} | {wr:.0f} | {f('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{f('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{f('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{f('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{f('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{int(r['launch__registers_per_thread'])} | {int(r['launch__grid_size'])} x {int(r['launch__block_size'])} |")


if __name__ == "__main__":
    main()
