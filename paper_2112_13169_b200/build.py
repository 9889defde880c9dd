"""In-tree native build: libvxm.so (sm_100a kernels + C-ABI) and libvoxmap_b200.so
(the C++ drop-in voxmap API over the C-ABI), plus the oracle builds used only
by tests and the CPU baseline. Everything lands inside the repo so it travels
to the GPU box with the snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: the reference forbids FMA contraction (-ffp-contract=off,
# proj/src/CMakeLists.txt:33-35); the kernels also spell every fp64 op with
# _rn intrinsics.
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-ffp-contract=off",
                  "-Xcompiler", "-Wall", f"-I{ROOT / 'include'}"]

CU_SOURCES = ["vxm_unity.cu"]
CU_INCLUDED = ["vxm_runtime.cu", "vxm_stages.cu"]
CU_HEADERS = ["vxm_device.cuh", "vxm_kernels.cuh", "vxm_aux_kernels.cuh", "vxm_tuning.h", "host/voxgrid_format.hpp"]


def _run(cmd, cwd=None):
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(map(str, cmd))}")
    return r.stdout + r.stderr


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_libvxm(force=False) -> Path:
    LIBDIR.mkdir(exist_ok=True)
    out = LIBDIR / "libvxm.so"
    deps = [CSRC / s for s in CU_SOURCES + CU_INCLUDED + CU_HEADERS] + [ROOT / "include" / "vxm.h"]
    if force or _stale(out, deps):
        objs = []
        for s in CU_SOURCES:
            o = LIBDIR / (Path(s).stem + ".o")
            _run([NVCC, *NVFLAGS, "-c", str(CSRC / s), "-o", str(o)])
            objs.append(str(o))
        _run([NVCC, *ARCH, "-shared", *objs, "-o", str(out)])
        for o in objs:
            os.remove(o)
    return out


HOST_CXX = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-ffp-contract=off",
            f"-I{ROOT / 'include'}", f"-I{ROOT / 'third_party' / 'eigen_subset'}"]


def build_dropin(force=False):
    """libvoxmap_b200.so: the C++ voxmap API (include/voxmap/) over libvxm.so,
    plus the C++ test driver tests/cpp/build/test_dropin."""
    lib = LIBDIR / "libvoxmap_b200.so"
    src = CSRC / "host" / "voxmap_api.cpp"
    fmt = CSRC / "host" / "voxgrid_format.hpp"
    hdrs = list((ROOT / "include" / "voxmap").rglob("*.hpp")) + [ROOT / "include" / "vxm.h"]
    if force or _stale(lib, [src, fmt, LIBDIR / "libvxm.so", *hdrs]):
        _run([*HOST_CXX, "-shared", str(src), f"-L{LIBDIR}", "-lvxm", "-Wl,-rpath,$ORIGIN", "-o", str(lib)])
    test_src = ROOT / "tests" / "cpp" / "test_dropin.cpp"
    test_bin = ROOT / "tests" / "cpp" / "build" / "test_dropin"
    if test_src.exists() and (force or _stale(test_bin, [test_src, lib, *hdrs])):
        test_bin.parent.mkdir(exist_ok=True)
        _run([*HOST_CXX, str(test_src), f"-L{LIBDIR}", "-lvoxmap_b200", "-lvxm",
              "-Wl,-rpath,$ORIGIN/../../../paper_2112_13169_b200/lib", "-o", str(test_bin)])
    return lib


def build_oracle(force=False):
    """oracle/_ref (reference sources) when /root/reference is present, and
    the plain-C restatement oracle/build/liboracle.so. Test infrastructure."""
    built = []
    c_src = ROOT / "oracle" / "voxmap_oracle.c"
    if c_src.exists():
        out = ROOT / "oracle" / "build" / "liboracle.so"
        out.parent.mkdir(exist_ok=True)
        if force or _stale(out, [c_src, ROOT / "oracle" / "voxmap_oracle.h"]):
            _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-Wall",
                  str(c_src), "-o", str(out), "-lm"])
        built.append(out)
    if Path("/root/reference/proj/src").exists():
        _run(["make", "-s", "-f", "oracle/Makefile.ref", f"-j{os.cpu_count() or 4}"], cwd=ROOT)
        built.append(ROOT / "oracle" / "_ref" / "libvoxmap_ref.so")
    return built


def build_ref_suites(force=False):
    """The reference's own unit-test programs (proj/tests/test_*.cpp,
    unmodified) against the drop-in headers and libvoxmap_b200.so
    (tests/cpp/Makefile.refsuites). Needs /root/reference: built here, the
    binaries travel to the GPU box. Test infrastructure."""
    if not Path("/root/reference/proj/tests").exists():
        return []
    _run(["make", "-s", "-f", "tests/cpp/Makefile.refsuites", f"-j{os.cpu_count() or 4}"]
         + (["-B"] if force else []), cwd=ROOT)
    return sorted((ROOT / "tests" / "cpp" / "build" / "ref_suites").glob("test_*[!.o]"))


def build_all(force=False):
    lib = build_libvxm(force)
    dropin = build_dropin(force)
    oracle = build_oracle(force)
    suites = build_ref_suites(force)
    return [lib, dropin, *oracle, *suites]


if __name__ == "__main__":
    for p in build_all(force="--force" in sys.argv):
        print(p)
