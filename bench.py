#!/usr/bin/env python
"""Benchmark of the alpha_{2,3} fill path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--fmt f64|u64|f32] [--engine auto|barrett|montgomery|fp64|staged|bulk|mixed|hybrid]
                    [--log2n 30] [--workload c2|c5] [--sweep FILE] [--ab FILE]

A "step" is one fill of 2^30 uniform doubles from seed
index a0 = 3^33+100 into device memory, per rank; rank r fills logical
offsets [r*2^30, (r+1)*2^30) (index sharding, no collective on the data path:
weak scaling). Rank 0 prints ONE JSON line.

* value      variates/s over all ranks, output resident in HBM, timed with CUDA
             events on the launching stream, max over ranks.
* sustained  the same step back to back for >= 1 s (the K-step headline is a
             burst shorter than the board power controller's window), clocks.
* e2e        the same metric through the public C-ABI call with a pinned HOST
             output (device generation + D2H inside the timed region);
             e2e_pageable: into a pageable numpy array.
* roofline   dominant kernel: algorithmic bytes written per launch
             (itemsize x 2^30) / average launch time vs the measured HBM peak.
* digest_verified_vs_oracle  the step's output digest (all ranks combined)
             against the oracle's committed digests of the same window.
* c5_strong  C5 (2^36 doubles index-sharded over the ranks, strong scaling),
             digest-verified, beside the C2 weak-scaling headline.
* cpu_baseline  the reference's own par::fill (oracle/_ref, compiled from
             /root/reference) on this host's cores, bounded sample (rank 0, N=1).

`--impl reference` times only the reference CPU implementation on the same
metric and config (rank 0; other ranks exit 0): one par::fill of the 2^30
window per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "uniform variates/sec & GB/s written vs HBM write peak, 1/2/4/8 B200"
UNIT = "variates/s"
A0 = 5559060566555523 + 100
FMT_ITEMSIZE = {"u64": 8, "f64": 8, "f32": 4}


def parse() -> argparse.Namespace:
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--fmt", default="f64", choices=["f64", "u64", "f32"])
    p.add_argument("--engine", default="auto")
    p.add_argument("--log2n", type=int, default=30)
    p.add_argument("--pace", type=float, default=None,
                   help="override the library's write-pacing target (GB/s; 0 = unpaced, <0 = automatic)")
    p.add_argument("--e2e-steps", type=int, default=0, help="host fills per e2e leg (0: min(steps, 20))")
    p.add_argument("--sustain-s", type=float, default=1.0, help="sustained window (s; 0 = off)")
    p.add_argument("--no-c5", action="store_true", help="skip the C5 strong-scaling section")
    p.add_argument("--c5-steps", type=int, default=5)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--sweep", default="", help="write a format x engine x size sweep (JSON lines)")
    p.add_argument("--ab", default="", help="interleaved engine A/B for --fmt, JSON lines to FILE")
    p.add_argument("--workload", default="c2", choices=["c2", "c5"],
                   help="c2: 2^log2n per GPU (weak scaling); c5: 2^36 total index-sharded (strong)")
    return p.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples: list[int] = []
        self.power: list[float] = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are best effort
            self.nvml = None

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                # instantaneous reading: the default power usage is a ~1 s average
                v = nv.nvmlDeviceGetFieldValues(self.h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
                if v.nvmlReturn == 0:
                    self.power.append(v.value.uiVal / 1000.0)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nvml:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self) -> dict:
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        limit = None
        try:
            limit = self.nvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0 if self.nvml else None
        except Exception:  # noqa: BLE001
            pass
        srt = sorted(self.samples)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_mhz_mean": statistics.mean(self.samples) if self.samples else None,
                "sm_mhz_p10": srt[len(srt) // 10] if srt else None,  # NVML's reading lags the power controller
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": names,
                "power_w_median": statistics.median(self.power) if self.power else None,  # instantaneous
                "power_limit_w": limit}


# --------------------------------------------------------------- workload
REF_WINDOW = 1 << 30  # the reference arm's per-step window (par::fill, parallel.cpp:101-105)


def workload(args, world: int) -> dict:
    """The `config` object of the JSON line. Both arms print exactly this dict
    (the reference arm on the same --fmt / --log2n / --workload / world)."""
    if args.workload == "c2":
        return {"workload": f"C2: fill 2^{args.log2n} {args.fmt} variates per GPU from seed index "
                            f"a0 = 3^33+100; rank r at base_offset r*2^{args.log2n} (weak scaling)",
                "items_per_step": world << args.log2n, "format": args.fmt, "layout": "contiguous",
                "seed_index": A0, "method": "BarrettModified"}
    return {"workload": f"C5: 2^36 {args.fmt} variates from seed index a0 = 3^33+100, index-sharded "
                        "over the GPUs (strong scaling)",
            "items_per_step": 1 << 36, "format": args.fmt, "layout": "contiguous",
            "seed_index": A0, "method": "BarrettModified"}


def golden_digest(fmt: str, start: int, count: int):
    """Digest of logical elements [start, start+count) of the a0 stream from the
    oracle's committed per-2^24-chunk table (tests/golden/chunk_digests.json,
    made and pinned by tests/golden/make_chunk_digests.py), or None when the
    window is not chunk-aligned or lies beyond the table."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "chunk_digests.json")) as f:
            g = json.load(f)
    except (OSError, ValueError):
        return None
    ch = 1 << g["chunk_log2"]
    rows = g["formats"].get(fmt, [])
    if start % ch or count % ch or (start + count) // ch > len(rows) or count == 0:
        return None
    s = ws = x = 0
    for r in rows[start // ch:(start + count) // ch]:
        s, ws, x = (s + int(r[0])) % (1 << 64), (ws + int(r[1])) % (1 << 64), x ^ int(r[2])
    return [s, ws, x]


def c5_golden():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "c5_digest.json")) as f:
            return [int(x) for x in json.load(f)["digest"]]
    except (OSError, ValueError, KeyError):
        return None


# ------------------------------------------------------------ reference arm
def reference_rate(n_sample: int, threads: int, reps: int = 1,
                   min_seconds: float = 0.0) -> tuple[float, float, int]:
    """Time the reference's par::fill (oracle/_ref) on `threads` workers over
    consecutive windows of the stream: at least `reps` calls and at least
    `min_seconds` of wall time. Returns (variates/s, seconds per call, calls)."""
    import numpy as np

    import oracle as O

    ref = O.Reference()
    out = np.empty(n_sample, dtype=np.float64)
    ref.fill(n_sample, O.FMT_F64, workers=threads, out=out)  # warm pages
    t0 = time.perf_counter()
    r = 0
    while r < reps or time.perf_counter() - t0 < min_seconds:
        ref.fill(n_sample, O.FMT_F64, workers=threads, base_offset=r * n_sample, out=out)
        r += 1
    dt = (time.perf_counter() - t0) / r
    return n_sample / dt, dt, r


def run_reference(args) -> None:
    """The reference arm: the unmodified reference par::fill (oracle/_ref, the
    /root/reference sources compiled in place) on every host thread, on this
    arm's config. Each step is one par::fill of the whole 2^30 window [0, 2^30)
    from a0 (the rank-0 shard of C2; a bounded 2^30 sample of the larger
    multi-GPU and C5 workloads)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import oracle as O

    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    config = workload(args, world)
    threads = os.cpu_count() or 1
    n_step = min(config["items_per_step"], REF_WINDOW)
    fmt = O.FMT_U64 if args.fmt == "u64" else O.FMT_F64  # the reference has no f32
    ref = O.Reference()
    out = np.empty(n_step, dtype=np.uint64 if fmt == O.FMT_U64 else np.float64)
    for _ in range(args.warmup):
        ref.fill(n_step, fmt, workers=threads, out=out)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.fill(n_step, fmt, workers=threads, out=out)
    dt = time.perf_counter() - t0
    value = n_step * args.steps / dt
    kind = "par::fill_residues" if fmt == O.FMT_U64 else "par::fill"
    sample = (f"{kind} of {n_step} {'residues' if fmt == O.FMT_U64 else 'doubles'} [0, 2^{n_step.bit_length() - 1}) "
              f"from a0 per step, W={threads} threads, Method::BarrettModified"
              + ("" if n_step == config["items_per_step"] else
                 f" (a 2^{n_step.bit_length() - 1} sample of the {config['items_per_step']}-item step)")
              + (" (f64: the reference has no f32 format)" if args.fmt == "f32" else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.workload == "c2" else "strong",
        "vs_baseline": None, "dtype": "u64" if fmt == O.FMT_U64 else "f64",
        "data": "synthetic: the generator has no inputs; output is the alpha_{2,3} stream",
        "config": config,
        "implementation": "reference C++ par::fill (oracle/_ref: unmodified /root/reference/proj/src "
                          "compiled -O3 -DNDEBUG) on the host cores",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gbs_written": value * 8 / 1e9,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
ENGINE_NAMES = {"auto": "Auto", "barrett": "Barrett", "montgomery": "Montgomery", "fp64": "FP64",
                "staged": "Staged", "bulk": "Bulk", "mixed": "Mixed",
                "hybrid": "Hybrid"}


def kernel_name(fmt: int, engine: int, paced: bool) -> str:
    """Template instance name of the dominant kernel for (format, engine)."""
    if paced and fmt != 2 and engine in (3, 6):  # FP64-pipe engines are paced
        return f"void k_fill_paced<{fmt}, {engine}, 0>(PacedArgs)"
    if engine == 4:
        return f"void k_fill_staged<{fmt}>(StagedArgs)"
    if engine == 5:
        return f"void k_fill_bulk<{fmt}, 3>(ContigArgs)"
    return f"void k_fill_contig<{fmt}, {engine}>(ContigArgs)"


def ncu_traffic(kernel: str, algorithmic_bytes: float) -> tuple[float | None, str | None]:
    """dram read+write bytes per launch of `kernel` from the committed
    `ncu --set full` summaries under profiles/ (tools/ncu_summary.py): of the
    captured launches of that kernel, the one whose size matches this launch
    (traffic closest to its algorithmic bytes; the capture also holds smaller
    launches of the same kernel)."""
    import glob

    best = None
    # Newest round first: its capture is of the code being measured.
    for rdir in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*")), reverse=True):
        if best is not None:
            break
        best = _ncu_best(kernel, algorithmic_bytes, sorted(glob.glob(os.path.join(rdir, "ncu_full_*.json"))))
    return (best[1], best[2]) if best else (None, None)


def _ncu_best(kernel: str, algorithmic_bytes: float, paths: list[str]):
    best = None
    for path in paths:
        try:
            with open(path) as f:
                rows = json.load(f)
        except (OSError, ValueError):
            continue
        for r in rows if isinstance(rows, list) else []:
            if r.get("kernel", "").strip() == kernel and "traffic_bytes" in r:
                d = abs(r["traffic_bytes"] - algorithmic_bytes)
                if best is None or d < best[0]:
                    best = (d, r["traffic_bytes"], os.path.relpath(path, ROOT))
    return best


def main() -> None:
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_1206_1187_b200 as B
    from paper_1206_1187_b200 import _lib, sharding
    from paper_1206_1187_b200 import build as bld

    bld.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # One process per GPU. BCN_DIST_BACKEND=gloo lets several ranks share one
    # GPU (NCCL refuses duplicate devices) so the multi-rank path can be
    # exercised on a single-GPU box; collectives then use CPU tensors.
    backend = os.environ.get("BCN_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    coll_dev = dev if backend == "nccl" else None
    # Under torchrun the process group is initialised even for one rank, so a
    # 1-GPU run exercises the same NCCL calls (digest all-gather, timing max)
    # as the 8-GPU one.
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if distributed:
        if backend == "nccl":
            # Communicator init lines on stderr (rank count, transports): the
            # only NCCL traffic is the 24-byte digest all-gather and the timing max.
            if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def barrier():
        if distributed:
            dist.barrier()

    if args.pace is not None:
        _, cps, mask = B.device.write_pacing_config()
        B.device.set_write_pacing(args.pace, cps, mask)
    fmt = B.Format[args.fmt.upper()]
    engine = B.Engine[ENGINE_NAMES[args.engine]]
    resolved = B.Engine(_lib.lib().bcn_auto_engine(int(fmt))) if engine == B.Engine.Auto else engine
    isz = FMT_ITEMSIZE[args.fmt]
    tdtype = {"f64": torch.float64, "u64": torch.int64, "f32": torch.float32}[args.fmt]
    stream = torch.cuda.current_stream(dev)
    lib = _lib.lib()
    config = workload(args, world)

    def rank_pieces(workload_name: str):
        """(base_offset, count) launches of this rank for one step."""
        if workload_name == "c2":
            n_rank = 1 << args.log2n
            start, count = sharding.shard(world * n_rank, world, rank)
            return start, count, [(start, count)]
        start, count = sharding.shard(1 << 36, world, rank)
        return start, count, list(sharding.chunks(start, count, 1 << 32))

    start, count, pieces = rank_pieces(args.workload)
    total_items = config["items_per_step"]
    scaling = "weak" if args.workload == "c2" else "strong"
    buf_items = max(c for _, c in pieces)
    buf = torch.empty(buf_items, dtype=tdtype, device=dev)
    raw = buf.view(torch.int64) if isz == 8 else buf.view(torch.int32)

    def make_step(pcs, out, f):
        plans = {c: B.par.make_plan(c, 1) for _, c in pcs}

        def step():
            for b, c in pcs:
                B.par.fill_format(out[:c], plans[c], A0, B.Method.BarrettModified, b, f,
                                  engine=engine, stream=stream)
        return step

    step = make_step(pieces, buf, fmt)

    def timed(fn, steps, warmup):
        """Per-call CUDA-event durations (ms), total ms and the number of our
        kernel launches for `steps` calls (after `warmup` untimed calls)."""
        for _ in range(warmup):
            fn()
        barrier()
        torch.cuda.synchronize(dev)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        lc0 = lib.bcn_launch_count()
        evs[0].record(stream)
        for i in range(steps):
            fn()
            evs[i + 1].record(stream)
        torch.cuda.synchronize(dev)
        launched = lib.bcn_launch_count() - lc0
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
        total = evs[0].elapsed_time(evs[-1])
        barrier()
        return per, total, launched

    def gather(vals: list[float]) -> list[list[float]]:
        """Every rank's `vals` (rank order)."""
        if not distributed:
            return [vals]
        t = torch.tensor(vals, dtype=torch.float64, device=coll_dev)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [o.tolist() for o in out]

    # Headline: device-resident fill, every step writes this rank's whole share.
    with ClockSampler(local) as clocks:
        per, my_ms, launches = timed(step, args.steps, args.warmup)
    total_ms = sharding.max_over_ranks(my_ms, coll_dev)
    value = total_items * args.steps / (total_ms * 1e-3)
    avg_step_ms = statistics.mean(per)
    launches_per_step = max(1, launches // args.steps)
    achieved_gbs = count * isz / (avg_step_ms * 1e-3) / 1e9  # this rank's kernel bytes / time

    # Sustained: back-to-back steps for >= --sustain-s seconds (the headline's
    # K steps are a burst shorter than the board power controller's window).
    sustained = None
    if args.sustain_s > 0:
        n_sus = max(args.steps, int(args.sustain_s * 1e3 / max(avg_step_ms, 1e-3)) + 1)
        with ClockSampler(local) as sclk:
            _, sus_ms, _ = timed(step, n_sus, 0)
        sus_ms = sharding.max_over_ranks(sus_ms, coll_dev)
        sustained = {"steps": n_sus, "seconds": sus_ms * 1e-3,
                     "value": total_items * n_sus / (sus_ms * 1e-3), "unit": UNIT,
                     "gbs_written": total_items * n_sus * isz / (sus_ms * 1e-3) / 1e9,
                     "clocks": sclk.summary()}
    per_rank = gather([my_ms / args.steps, achieved_gbs])

    # Constant writer (the paper's memory ceiling) with the identical pattern,
    # measured after the headline so its power draw does not precede it.
    const_per, _, _ = timed(lambda: B.device.fill_constant(raw, stream=stream),
                            max(20, args.steps // 4), 5)
    const_gbs = buf_items * isz / (statistics.mean(const_per) * 1e-3) / 1e9
    pace_now = B.device.write_pacing_config()
    lib.bcn_set_write_pacing(0.0, pace_now[1], pace_now[2])
    const_per_u, _, _ = timed(lambda: B.device.fill_constant(raw, stream=stream),
                              max(20, args.steps // 4), 5)
    lib.bcn_set_write_pacing(*pace_now)
    # The same paced writer with random words: toggles the HBM interface like
    # real output (a constant pattern draws ~230 W less at 7 TB/s), so under
    # the board power cap this is the realistic write ceiling.
    noise_per, _, _ = timed(lambda: B.device.fill_noise(raw, stream=stream), args.steps, 5)
    noise_gbs = buf_items * isz / (statistics.mean(noise_per) * 1e-3) / 1e9
    const_unpaced_gbs = buf_items * isz / (statistics.mean(const_per_u) * 1e-3) / 1e9

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (STREAM copy, measured)" if "hbm_gbs" in peaks \
        else "fallback 6.65 TB/s (B200_PROFILING.md)"

    # Verification (untimed): digest of every launch's output, combined over
    # the shards with a 24-byte all-gather (the only collective), against the
    # oracle's digests of the same window.
    def verify(pcs, out, out_raw, f, want):
        parts = []
        for b, c in pcs:
            B.par.fill_format(out[:c], B.par.make_plan(c, 1), A0, B.Method.BarrettModified, b, f,
                              engine=engine, stream=stream)
            parts.append(B.device.digest(out_raw[:c], index_base=b))
        local_d = sharding.combine(parts)
        glob = sharding.allgather_digest(local_d, coll_dev) if distributed else local_d
        return glob, (None if want is None else list(glob) == list(want))

    want = golden_digest(args.fmt, 0, total_items) if args.workload == "c2" else \
        (c5_golden() if args.fmt == "f64" else None)
    global_digest, verified = verify(pieces, buf, raw, fmt, want)

    # End to end through the public API into HOST memory, D2H inside the timed
    # region: a pinned buffer (`e2e`) and a pageable numpy array (`e2e_pageable`,
    # the reference user's std::vector-backed span, parallel.hpp:48-49).
    e2e = e2e_pageable = None
    e2e_steps = args.e2e_steps or min(args.steps, 20)
    if not args.no_e2e and args.workload == "c2":
        import numpy as np

        hplan = B.par.make_plan(count, 1)

        def host_rate(host):
            B.par.fill_format(host, hplan, A0, B.Method.BarrettModified, start, fmt, engine=engine)
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                B.par.fill_format(host, hplan, A0, B.Method.BarrettModified, start, fmt, engine=engine)
            dt = sharding.max_over_ranks(time.perf_counter() - t0, coll_dev)
            barrier()
            return dt

        host = torch.empty(count, dtype=tdtype, pin_memory=True)
        dt = host_rate(host)
        # The e2e roofline: a plain D2H copy of the same bytes into the same
        # pinned buffer (PCIe bound), timed the same way.
        src = buf[:count]
        host.copy_(src)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            host.copy_(src)
        torch.cuda.synchronize(dev)
        d2h_gbs = count * isz * e2e_steps / (time.perf_counter() - t0) / 1e9
        e2e_gbs = count * isz * e2e_steps / dt / 1e9
        e2e = {"value": total_items * e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": count * isz, "steps": e2e_steps,
               "gbs_delivered": e2e_gbs, "d2h_copy_gbs": d2h_gbs, "frac_of_d2h_copy": e2e_gbs / d2h_gbs,
               "note": "bcn_fill with a pinned host pointer: chunked device generation + D2H on "
                       "two streams; inputs are scalar kernel arguments (seed index, offset, "
                       "count), so there is no H2D buffer"}
        del host
        pageable = np.empty(count, dtype={"f64": np.float64, "u64": np.uint64, "f32": np.float32}[args.fmt])
        dt = host_rate(pageable)
        e2e_pageable = {"value": total_items * e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": count * isz, "steps": e2e_steps,
                        "gbs_delivered": count * isz * e2e_steps / dt / 1e9,
                        "note": "bcn_fill into a pageable numpy array (the reference's std::vector "
                                "case): device chunks -> pinned staging -> host copy pool"}
        del pageable

    # C5 strong scaling beside the C2 weak-scaling headline: 2^36 f64 from a0,
    # index-sharded over the ranks, digest-verified against the oracle.
    c5 = None
    if args.workload == "c2" and not args.no_c5:
        del buf, raw
        torch.cuda.empty_cache()
        s5, n5 = sharding.shard(1 << 36, world, rank)
        p5 = list(sharding.chunks(s5, n5, 1 << 32))
        buf5 = torch.empty(max(c for _, c in p5), dtype=torch.float64, device=dev)
        step5 = make_step(p5, buf5, B.Format.F64)  # the C5 digest is of doubles
        per5, ms5, l5 = timed(step5, args.c5_steps, 2)
        ms5 = sharding.max_over_ranks(ms5, coll_dev)
        d5, ok5 = verify(p5, buf5, buf5.view(torch.int64), B.Format.F64, c5_golden())
        c5 = {"workload": workload(argparse.Namespace(workload="c5", fmt="f64", log2n=36), world)["workload"],
              "items_per_step": 1 << 36, "n_gpus": world, "steps": args.c5_steps, "warmup": 2,
              "ms_per_step": ms5 / args.c5_steps, "value": (1 << 36) * args.c5_steps / (ms5 * 1e-3),
              "unit": UNIT, "scaling": "strong", "gpu_launches": int(l5),
              "gbs_written": (1 << 36) * 8 * args.c5_steps / (ms5 * 1e-3) / 1e9,
              "digest": [str(x) for x in d5], "digest_verified_vs_oracle": ok5}
        del buf5

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        # Bounded sample of the C2 workload: consecutive 2^27-double windows of
        # the stream for >= 10 s of wall time on every host thread.
        rate, secs, calls = reference_rate(1 << 27, threads, min_seconds=10.0)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": f"reference par::fill (oracle/_ref = unmodified /root/reference sources, "
                         f"g++ -O3): {calls} consecutive windows of 2^27 doubles of the C2 stream, "
                         f"W={threads} threads, {calls * secs:.2f} s wall"}
        # the single-thread rate too (config 1 = 10^6 doubles,
        # repeated over consecutive windows for >= 2 s).
        rate1, secs1, calls1 = reference_rate(10**6, 1, reps=5, min_seconds=2.0)
        cpu["single_thread"] = {"value": rate1, "unit": UNIT, "cores": 1,
                                "sample": f"config 1 windows: {calls1} x par::fill of 10^6 doubles, W=1, "
                                          f"{calls1 * secs1:.2f} s"}

    if args.ab or args.sweep:
        buf = torch.empty(buf_items, dtype=tdtype, device=dev)
    ab_rows = run_ab(B, torch, dev, stream, timed, buf, fmt, args.ab) if args.ab else []
    sweep_rows = run_sweep(B, dev, stream, timed) if args.sweep else []

    if rank == 0:
        pace, pace_src = B.device.device_write_pacing(local)
        kname = kernel_name(int(fmt), int(resolved), pace > 0)
        bytes_per_launch = count * isz / launches_per_step
        traffic, traffic_src = ncu_traffic(kname, bytes_per_launch)
        ceiling = max(const_gbs, noise_gbs)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": args.fmt,
            "data": "synthetic: the generator has no inputs; output is the alpha_{2,3} stream",
            "config": config,
            "launch": {"engine": B.par.Engine(resolved).name,
                       "write_pacing_gbs": pace if (pace > 0 and isz == 8) else None,
                       "write_pacing_source": pace_src,
                       "pace_calibration": [[t, round(a, 1)] for t, a in B.device.pace_calibration(local)],
                       "write_pacing_ctas_per_sm": B.device.write_pacing_config()[1],
                       "parallelism": f"index-sharded x{world}, no data-path collective",
                       "l2": f"output {buf_items * isz / 2**30:.0f} GiB per launch >> 126 MB L2 "
                             "(outputs larger than L2, no flush needed)"},
            "gbs_written": value * isz / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                         "frac": achieved_gbs / peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src, "kernel": kname,
                         "bytes_per_launch": bytes_per_launch,
                         "algorithmic_bytes_per_variate": isz,
                         "avg_launch_ms": avg_step_ms / launches_per_step,
                         "write_ceiling_gbs": ceiling,
                         "frac_of_write_ceiling": achieved_gbs / ceiling,
                         "constant_writer_gbs": const_gbs,
                         "constant_writer_unpaced_gbs": const_unpaced_gbs,
                         "frac_of_constant_writer": achieved_gbs / const_gbs,
                         "noise_writer_gbs": noise_gbs,
                         "frac_of_noise_writer": achieved_gbs / noise_gbs,
                         "note": "peak = measured STREAM copy (read+write bytes), the contract's "
                                 "denominator; a write-only stream exceeds it on this part, so frac "
                                 "can exceed 1. frac_of_write_ceiling divides by the faster of the "
                                 "paced Constant / noise writers measured in this run (same "
                                 "geometry, no arithmetic)"},
            "sustained": sustained,
            "per_rank": [{"rank": r, "ms_per_step": v[0], "gbs": v[1]} for r, v in enumerate(per_rank)],
            "e2e": e2e,
            "e2e_pageable": e2e_pageable,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "digest": [str(x) for x in global_digest],
            "digest_verified_vs_oracle": verified,
            "c5_strong": c5,
        }
        for name, rows in (("ab_file", ab_rows), ("sweep_file", sweep_rows)):
            if rows:
                path = args.ab if name == "ab_file" else args.sweep
                with open(path, "w") as f:
                    for r in rows:
                        f.write(json.dumps(r) + "\n")
                line[name] = path
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def run_ab(B, torch, dev, stream, timed, buf, fmt, path) -> list[dict]:
    """Interleaved A/B of every engine for one format: 15 rounds x 6 launches
    each, round-robin, so drift affects all engines alike."""
    plan = B.par.make_plan(buf.numel(), 1)
    engines = [e for e in B.Engine if e != B.Engine.Auto]
    times = {e.name: [] for e in engines}
    times["Constant"] = []
    raw = buf.view(torch.int64) if buf.element_size() == 8 else buf.view(torch.int32)
    for _ in range(15):
        for e in engines:
            per, _, _ = timed(lambda: B.par.fill_format(buf, plan, A0, B.Method.BarrettModified, 0,
                                                        fmt, engine=e, stream=stream), 6, 1)
            times[e.name] += per
        per, _, _ = timed(lambda: B.device.fill_constant(raw, stream=stream), 6, 1)
        times["Constant"] += per
    nbytes = buf.numel() * buf.element_size()
    rows = []
    for k, v in times.items():
        med = statistics.median(v)
        rows.append({"fmt": B.Format(fmt).name, "engine": k, "median_ms": med, "min_ms": min(v),
                     "gbs_median": nbytes / (med * 1e-3) / 1e9, "samples": len(v)})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    return rows


def run_sweep(B, dev, stream, timed) -> list[dict]:
    """formats x engines x sizes 2^28..2^32, device-resident."""
    import torch

    rows = []
    for log2n in (28, 29, 30, 31, 32):
        for fmt in ("u64", "f64", "f32"):
            isz = FMT_ITEMSIZE[fmt]
            nbytes = (1 << log2n) * isz
            tdt = {"f64": torch.float64, "u64": torch.int64, "f32": torch.float32}[fmt]
            out = torch.empty(1 << log2n, dtype=tdt, device=dev)
            plan = B.par.make_plan(1 << log2n, 1)
            f = B.Format[fmt.upper()]
            for e in [e for e in B.Engine if e != B.Engine.Auto]:
                per, _, _ = timed(lambda: B.par.fill_format(out, plan, A0, B.Method.BarrettModified,
                                                            0, f, engine=e, stream=stream), 10, 3)
                ms = statistics.median(per)
                rows.append({"log2n": log2n, "fmt": fmt, "engine": e.name, "ms": ms,
                             "gbs": nbytes / (ms * 1e-3) / 1e9,
                             "gvariates_s": (1 << log2n) / (ms * 1e-3) / 1e9})
                print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            raw = out.view(torch.int32) if isz == 4 else out.view(torch.int64)
            per, _, _ = timed(lambda: B.device.fill_constant(raw, stream=stream), 10, 3)
            ms = statistics.median(per)
            rows.append({"log2n": log2n, "fmt": fmt, "engine": "Constant", "ms": ms,
                         "gbs": nbytes / (ms * 1e-3) / 1e9})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del out
    return rows


if __name__ == "__main__":
    main()
