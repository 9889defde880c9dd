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
