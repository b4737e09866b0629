"""The C++ drop-in: include/bcnrand/*.hpp keep the reference's API over the C
ABI. Two programs written against those headers are built by tests/cpp/Makefile:

* tests/cpp/build/test_dropin — this repo's C++ tests of the drop-in;
* oracle/_ref/ref_tests_on_b200 — the REFERENCE's own unit tests
  (tests/test_{generator,parallel,quality,selftest,bench,cli}.cpp, unmodified,
  compiled in place from /root/reference) linked against libbcnrand_b200.so,
  i.e. the reference's test suite running on the B200 library (GPU);
* oracle/_ref/ref_host_tests — its tests/test_{modred,oracle}.cpp against the
  host-only parts of the drop-in (CPU suite).
"""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")
REFTESTS = os.path.join(ROOT, "oracle", "_ref", "ref_tests_on_b200")
DEVICE_API = os.path.join(ROOT, "tests", "cpp", "build", "test_device_api")


REF_HOST = os.path.join(ROOT, "oracle", "_ref", "ref_host_tests")
CMAKE_DIR = os.path.join(ROOT, "build", "cmake")
CMAKE_DROPIN = os.path.join(CMAKE_DIR, "bcn_test_dropin")


def test_cmake_target_bcnrand_core_builds():
    """CMakeLists.txt exports the reference's target name `bcnrand_core`
    (reference src/CMakeLists.txt): configure + build the library for sm_100a
    and a program linked only against `bcnrand_core`, as a reference user's
    CMake project would."""
    cmake = shutil.which("cmake")
    if cmake is None:
        pytest.skip("cmake not installed")
    os.makedirs(CMAKE_DIR, exist_ok=True)
    env = dict(os.environ, CUDACXX=os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"))
    gen = ["-G", "Ninja"] if shutil.which("ninja") else []
    r = subprocess.run([cmake, "-S", ROOT, "-B", CMAKE_DIR, *gen, "-DBCN_BUILD_TESTS=ON"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    r = subprocess.run([cmake, "--build", CMAKE_DIR, "-j", "8"], capture_output=True, text=True,
                       env=env, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert os.path.exists(CMAKE_DROPIN)
    elf = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(CMAKE_DIR, "libbcnrand_b200.so")], capture_output=True, text=True)
    if elf.returncode == 0:
        assert "sm_100a" in elf.stdout and "sm_52" not in elf.stdout, elf.stdout


def test_reference_host_tests_pass_on_the_dropin():
    """The reference's own tests/test_modred.cpp (goldens, exhaustive and random
    agreement of all four step kernels with reduce_ref, preconditions, the
    constant-table self-check with corrupted tables) and tests/test_oracle.cpp
    (the alpha-series expansion equals seed_from_index, period law, orders),
    compiled unmodified against include/bcnrand/{modred,oracle,generator}.hpp.
    Host-only: runs without a GPU."""
    if os.path.isdir("/root/reference/proj"):
        r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "ref"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    if not os.path.exists(REF_HOST):
        pytest.skip("oracle/_ref/ref_host_tests not built and /root/reference absent")
    r = subprocess.run([REF_HOST], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_device_api_arithmetic_on_host():
    """include/bcnrand_device.cuh compiled as plain C++: the Barrett mulmod
    against exact 128-bit arithmetic (edges + 2e7 random pairs), the step,
    skip-ahead composition and the reference goldens — no GPU involved."""
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "device_host"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "build", "test_device_api_host")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "[device-api-host] ok" in r.stdout, r.stdout + r.stderr


def test_dropin_headers_compile_and_link(bcn):
    """Builds against the headers + product library here (no GPU needed)."""
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "dropin"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert os.path.exists(DROPIN)
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "device"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    if os.path.isdir("/root/reference/proj"):
        r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "ref"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def _run(path: str) -> str:
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "| 0 failed" in out
    return out


CLI = os.path.join(ROOT, "tests", "cpp", "build", "bcnrand")


def test_cli_executable_usage_paths():
    """The `bcnrand` executable (include/bcnrand/cli.hpp, tools/bcnrand_main.cpp):
    the paths that need no GPU — seed-info and the usage / I/O exit codes of
    the reference (cli.cpp:24-27, test_cli.cpp:127-143)."""
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "cli"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

    def run(*args):
        return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=60)

    r = run("seed-info", "5559060566555623")
    assert r.returncode == 0 and "z0             = 4258649398211344" in r.stdout
    assert "z0 * 3^-33     = 0.76607357434316758" in r.stdout
    assert run("seed-info", "5559060566555622").returncode == 2
    assert run("seed-info", "9007199254740992").returncode == 0
    assert run("seed-info", "9007199254740993").returncode == 2
    assert run("gen", "--n", "5", "--seed", "100").returncode == 2
    assert run("gen", "--n", "5", "--format", "xml").returncode == 2
    assert run("gen").returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("gen", "--n", "5", "--out", "/nonexistent-dir/x").returncode == 3
    assert run("gen", "--n", "5", "--bogus", "1").returncode == 2
    assert run("--help").returncode == 0


@pytest.mark.gpu
def test_cli_executable_generates(cuda, tmp_path):
    """`bcnrand gen` on the GPU: raw-u64 n=1 is the golden z1, raw-f64 bytes are
    identical for W = 1 / 8 / 8 interleaved and chunked streaming, and
    `selftest --fast` passes."""
    if not os.path.exists(CLI):
        pytest.skip("tests/cpp/build/bcnrand not built")
    one = tmp_path / "one.u64"
    assert subprocess.run([CLI, "gen", "--n", "1", "--format", "raw-u64", "--out", str(one)]).returncode == 0
    assert int.from_bytes(one.read_bytes(), "little") == 2138759898642167
    outs = []
    for extra in ([], ["--workers", "8"], ["--workers", "8", "--layout", "interleaved"], ["--chunk", "7777"]):
        f = tmp_path / f"u{len(outs)}.f64"
        assert subprocess.run([CLI, "gen", "--n", "40000", "--format", "raw-f64", "--out", str(f), *extra]).returncode == 0
        outs.append(f.read_bytes())
    assert len(outs[0]) == 320000 and all(o == outs[0] for o in outs)
    r = subprocess.run([CLI, "selftest", "--fast"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "selftest: all checks passed" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_suite(cuda):
    if not os.path.exists(DROPIN):
        pytest.skip("tests/cpp/build/test_dropin not built")
    _run(DROPIN)


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_b200_library(cuda):
    """The reference's test_generator.cpp / test_parallel.cpp / test_quality.cpp /
    test_selftest.cpp / test_bench.cpp / test_cli.cpp (49 cases, ~3.5M
    assertions incl. worker/layout invariance, base_offset windows, the
    built-in selftest with a corrupted constant table, the throughput harness
    and the `bcnrand` command line: byte formats, chunked == single-shot,
    exit codes) pass when compiled against the drop-in headers and run on the
    GPU."""
    if not os.path.exists(REFTESTS):
        pytest.skip("oracle/_ref/ref_tests_on_b200 not built (needs /root/reference at build time)")
    out = _run(REFTESTS)
    assert "test cases: 49 | 49 passed | 0 failed" in out, out


@pytest.mark.gpu
def test_cmake_built_dropin_suite(cuda):
    """The drop-in test program built through CMakeLists.txt's `bcnrand_core`
    target (and its own libbcnrand_b200.so) passes on the GPU."""
    if not os.path.exists(CMAKE_DROPIN):
        pytest.skip("build/cmake/bcn_test_dropin not built")
    _run(CMAKE_DROPIN)


@pytest.mark.gpu
def test_device_side_api_matches_library_fill(cuda):
    """include/bcnrand_device.cuh inside a user kernel == bcn_fill, bit for bit."""
    if not os.path.exists(DEVICE_API):
        pytest.skip("tests/cpp/build/test_device_api not built")
    r = subprocess.run([DEVICE_API], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[device-api] ok" in r.stdout
