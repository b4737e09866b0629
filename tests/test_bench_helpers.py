"""CPU checks of bench.py's bookkeeping (no GPU): the roofline's kernel name
and ncu traffic lookup, the reference arm's JSON line, and the shard plan of
the C5 workload."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1206_1187_b200 import sharding  # noqa: E402


def test_kernel_name_follows_the_launch_choice():
    # FP64-pipe engines are paced for the 8-byte formats; f32 and the integer
    # engines run the unpaced persistent kernel; bulk / staged have their own.
    assert bench.kernel_name(1, 3, True) == "void k_fill_paced<1, 3, 0>(PacedArgs)"
    assert bench.kernel_name(0, 6, True) == "void k_fill_paced<0, 6, 0>(PacedArgs)"
    assert bench.kernel_name(2, 3, True) == "void k_fill_contig<2, 3>(ContigArgs)"
    assert bench.kernel_name(1, 1, True) == "void k_fill_contig<1, 1>(ContigArgs)"
    assert bench.kernel_name(1, 3, False) == "void k_fill_contig<1, 3>(ContigArgs)"
    assert bench.kernel_name(1, 4, True) == "void k_fill_staged<1>(StagedArgs)"
    assert bench.kernel_name(1, 5, True) == "void k_fill_bulk<1, 3>(ContigArgs)"


def test_ncu_traffic_picks_the_size_matched_launch():
    """The committed capture holds the headline kernel at 2^30 and at 2^28
    items; the bench must read the 8 GiB launch for an 8 GiB step."""
    t, src = bench.ncu_traffic("void k_fill_paced<1, 3, 0>(PacedArgs)", 8 * 2**30)
    assert src and src.startswith("profiles/")
    assert abs(t - 8 * 2**30) / (8 * 2**30) < 0.02
    t_small, _ = bench.ncu_traffic("void k_fill_paced<1, 3, 0>(PacedArgs)", 8 * 2**28)
    assert abs(t_small - 8 * 2**28) / (8 * 2**28) < 0.05
    assert bench.ncu_traffic("no such kernel", 1.0) == (None, None)


def test_c5_launch_plan_covers_2_36_at_every_world_size():
    for world in (1, 2, 4, 8):
        covered = 0
        for r in range(world):
            start, count = sharding.shard(1 << 36, world, r)
            pieces = list(sharding.chunks(start, count, 1 << 32))
            assert all(c <= 1 << 32 for _, c in pieces)
            assert sum(c for _, c in pieces) == count
            covered += count
        assert covered == 1 << 36


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj") and
                    not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbcnref.so")),
                    reason="reference library unavailable")
def test_reference_arm_line_is_complete():
    """`bench.py --impl reference` prints one JSON line with the contract keys
    (tiny run: 2 steps of a 2^20 sample)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--log2n", "20"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1


def test_cpu_baseline_sample_is_time_bounded():
    """cpu_baseline times consecutive windows of the stream until a minimum
    wall time has passed (the 10 s sample of the bench line), and at least
    `reps` calls."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbcnref.so")):
        pytest.skip("oracle/_ref not built")
    rate, secs, calls = bench.reference_rate(1 << 16, 2, min_seconds=0.2)
    assert rate > 0 and calls * secs >= 0.2
    rate, secs, calls = bench.reference_rate(1 << 10, 1, reps=3)
    assert calls >= 3
