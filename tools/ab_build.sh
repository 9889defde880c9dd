#!/bin/bash
# Scratch A/B: build lib/libvxm_<tag>.so with extra nvcc defines, e.g.
#   tools/ab_build.sh mul -DVXM_FAST_MUL=1 ; VXM_LIB_NAME=libvxm_mul.so python tools/quick_time.py
set -e
tag=$1; shift
cd "$(dirname "$0")/.."
python - "$tag" "$@" <<'PY'
import sys
from paper_2112_13169_b200 import build as b
tag, defs = sys.argv[1], sys.argv[2:]
o = b.LIBDIR / f"vxm_{tag}.o"
b._run([b.NVCC, *b.NVFLAGS, *defs, "-c", str(b.CSRC / "vxm_unity.cu"), "-o", str(o)])
b._run([b.NVCC, *b.ARCH, "-shared", str(o), "-o", str(b.LIBDIR / f"libvxm_{tag}.so")])
o.unlink()
PY
