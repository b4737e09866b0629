"""The `gen` byte formats (reference cli.cpp:79-147), mirroring the cases of
the reference's tests/test_cli.cpp on the GPU path."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
from paper_1206_1187_b200 import cli


def run(*args) -> int:
    return cli.main(list(args))


def test_usage_and_io_errors_before_device_work(tmp_path):
    """test_cli.cpp:127-133 (exit 2 usage, 3 I/O) — validated before any fill."""
    assert run("gen", "--n", "5", "--seed", "100") == 2
    assert run("gen", "--n", "5", "--format", "xml") == 2
    assert run("gen") == 2
    assert run("frobnicate") == 2
    assert run("gen", "--n", "5", "--out", "/nonexistent-dir/x") == 3
    assert run("gen", "--n", "0") == 2
    assert run("gen", "--n", "5", "--method", "mt19937") == 2


def test_text_formatter_is_printf_17g(bcn):
    v = np.array([0.1, 1.0 / 3.0, 5e-17, 0.999999999999999889, 0.38473405228023527])
    assert cli.format_text(v) == b"".join(b"%.17g\n" % x for x in v)


@pytest.mark.gpu
def test_gen_formats_match_reference_cases(bcn, cuda, oracle, tmp_path):
    # test_cli.cpp:76-86: raw-u64 n=1 is the first iterate, little endian
    one = tmp_path / "one.u64"
    assert run("gen", "--n", "1", "--seed", "5559060566555623", "--format", "raw-u64",
               "--out", str(one)) == 0
    assert int.from_bytes(one.read_bytes(), "little") == 2138759898642167
    # :44-74: text lines parse to the exact doubles and round-trip at %.17g
    txt = tmp_path / "t.txt"
    assert run("gen", "--n", "200", "--format", "text", "--out", str(txt)) == 0
    vals = [float(x) for x in txt.read_text().split()]
    assert vals == list(oracle.fill(200, O.FMT_F64))
    assert all(0.0 < v < 1.0 for v in vals)
    # :88-103: byte-identical across W and layouts (interleaved is de-interleaved)
    files = []
    for extra in ([], ["--workers", "8"], ["--workers", "8", "--layout", "interleaved"]):
        f = tmp_path / f"w{len(files)}.f64"
        assert run("gen", "--n", "40000", "--format", "raw-f64", *extra, "--out", str(f)) == 0
        files.append(f.read_bytes())
    assert files[0] == files[1] == files[2]
    assert files[0] == oracle.fill(40000, O.FMT_F64).tobytes()
    # :105-114: methods give identical files; :116-125 chunked == single shot
    a, b = tmp_path / "a.f64", tmp_path / "b.f64"
    assert run("gen", "--n", "30000", "--format", "raw-f64", "--method", "Ref128", "--out", str(a)) == 0
    assert run("gen", "--n", "30000", "--format", "raw-f64", "--method", "LEcuyer", "--chunk", "7777",
               "--out", str(b)) == 0
    assert a.read_bytes() == b.read_bytes()
    # --keep-physical emits the interleaved buffer as is
    k = tmp_path / "k.u64"
    assert run("gen", "--n", "1000", "--format", "raw-u64", "--workers", "7", "--layout",
               "interleaved", "--keep-physical", "--out", str(k)) == 0
    phys = np.frombuffer(k.read_bytes(), dtype="<u8")
    assert np.array_equal(phys, oracle.fill(1000, O.FMT_U64, workers=7, layout=O.INTERLEAVED))
    assert run("seed-info", "9007199254740993") == 2 and run("seed-info", "9007199254740992") == 0
    assert not os.path.exists(tmp_path / "missing")
