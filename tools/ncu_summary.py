#!/usr/bin/env python
"""Summarise ncu reports into small JSON files for profiles/ (the .ncu-rep
binaries stay out of git).

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] -o profiles/r01/ncu_x.json
    python tools/ncu_summary.py --launches gpurun_out/launches.csv -o profiles/r01/launches.json
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__sectors_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_op_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second",
    "dram__cycles_elapsed.avg.per_second",
    "smsp__average_warp_latency_issue_stalled_lg_throttle",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_drain",
]


def summarise_report(path: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"report": path.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = vals[i].replace(",", "")
                try:
                    d[m] = float(v)
                except ValueError:
                    d[m] = v
                d[m + ".unit"] = units[i]
        if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = d["dram__bytes_read.sum"] * scale.get(d["dram__bytes_read.sum.unit"], 1)
            wr = d["dram__bytes_write.sum"] * scale.get(d["dram__bytes_write.sum.unit"], 1)
            d["traffic_bytes"] = rd + wr
        res.append(d)
    return res


def summarise_launches(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())

    def entry(v):
        # A kernel may run at several sizes in one command (e.g. the bench's
        # full-size fills and its 64 MiB host-output chunks): `large` holds
        # the launches within 2x of the longest one.
        big = [x for x in v if x >= 0.5 * max(v)]
        return {"launches": len(v), "sum_ns": sum(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot,
                "large": {"launches": len(big), "mean_ns": sum(big) / len(big), "min_ns": min(big),
                          "max_ns": max(big)}}

    return {"source": path.split("/")[-1], "unit": "ns", "kernels": {k: entry(v) for k, v in agg.items()}}


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("reports", nargs="*")
    p.add_argument("--launches", default="")
    p.add_argument("-o", "--out", required=True)
    a = p.parse_args()
    data = summarise_launches(a.launches) if a.launches else [r for f in a.reports for r in summarise_report(f)]
    with open(a.out, "w") as f:
        json.dump(data, f, indent=1)
    print(a.out)


if __name__ == "__main__":
    main()
