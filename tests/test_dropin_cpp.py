"""Runs the C++ drop-in API driver (tests/cpp/test_dropin.cpp, built by
build()) on the GPU: the reference's unit cases compiled against
include/voxmap/ and linked to libvoxmap_b200.so -> libvxm.so."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "build" / "test_dropin"


@pytest.mark.gpu
def test_dropin_cpp_cases(gpu_lib):
    if not BIN.exists():
        pytest.fail(f"{BIN} not built (run __graft_entry__.build())")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_dropin_binary_links_the_gpu_library():
    # CPU-side check: the driver resolves its voxmap symbols from the in-tree libraries
    if not BIN.exists():
        pytest.skip("not built")
    out = subprocess.run(["ldd", str(BIN)], capture_output=True, text=True).stdout
    assert "libvoxmap_b200.so" in out and "libvxm.so" in out and "not found" not in out


# The reference's OWN unit-test programs (proj/tests/test_*.cpp, compiled
# unmodified by tests/cpp/Makefile.refsuites against include/voxmap, the
# Eigen subset and a doctest stand-in, linked to libvoxmap_b200.so).
SUITES = ("test_kernels", "test_integrator", "test_raytracer", "test_grid_core", "test_geometry", "test_pipeline")
SUITE_DIR = Path(__file__).resolve().parent / "cpp" / "build" / "ref_suites"


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_on_b200(gpu_lib, suite):
    exe = SUITE_DIR / suite
    if not exe.exists():
        pytest.fail(f"{exe} not built (make -f tests/cpp/Makefile.refsuites, run by build() here)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "| 0 failed" in r.stdout, r.stdout


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_links_the_gpu_library(suite):
    exe = SUITE_DIR / suite
    if not exe.exists():
        pytest.skip("not built")
    out = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
    assert "libvoxmap_b200.so" in out and "libvxm.so" in out and "not found" not in out
    assert "libvoxmap_ref" not in out  # the product library, not the oracle build


def test_reference_acceptance_reproduces_recorded_run():
    """oracle/_ref/acceptance (proj/tests/acceptance.cpp compiled unmodified
    against the reference sources) prints the recorded run
    (proj/test_output.txt:21-33, committed as tests/golden/acceptance_recorded.txt)
    line for line, timings aside: 11 PASS and criterion 9 FAIL with the Free
    counts 29712 / 28900 / 32613 / 39082."""
    import re

    exe = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "acceptance"
    if not exe.exists():
        pytest.skip("oracle/_ref not built")
    strip = lambda s: [re.sub(r" \(\d+\.\d+ s\)", "", ln) for ln in s.strip().splitlines()]  # noqa: E731
    want = strip((Path(__file__).resolve().parent / "golden" / "acceptance_recorded.txt").read_text())
    # criteria 8 (log-log slope of wall times) and 10 (a 3x wall-time ratio)
    # measure this host's timings, so a busy host can flip their verdict: their
    # text must match with either verdict, every other line exactly (a few runs
    # are tried for the exact recorded output first)
    timed = ("] 8: ", "] 10: ")
    untag = lambda ln: re.sub(r"^\[(PASS|FAIL)\] ", "", ln)  # noqa: E731
    for _ in range(3):
        r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
        got = strip(r.stdout)
        if got == want:
            break
    assert r.returncode == 1  # the recorded run fails criterion 9 too
    assert len(got) == len(want)
    for g, w in zip(got[:-1], want[:-1]):
        if any(t in w for t in timed):
            assert untag(g) == untag(w), (g, w)
        else:
            assert g == w, (g, w)
    extra = sum(1 for g in got if g.startswith("[FAIL]") and any(t in g for t in timed))
    assert got[-1] == f"acceptance: {1 + extra} of 12 criteria failed", got[-1]
