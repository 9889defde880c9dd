#!/bin/bash
# Build lib/libvxm_<tag>.so from a git revision (default HEAD) for same-box
# A/B timing against the working tree: tools/build_rev_lib.sh [rev] [tag]
set -e
rev=${1:-HEAD}; tag=${2:-head}
cd "$(dirname "$0")/.."
root=$(pwd)
wt=$(mktemp -d /tmp/vxmrev.XXXX)
git worktree add -f "$wt" "$rev" -q
(cd "$wt" && python - "$root" "$tag" <<'PY'
import sys
root, tag = sys.argv[1], sys.argv[2]
sys.path.insert(0, '.')
from paper_2112_13169_b200 import build as b
o = f"/tmp/vxm_{tag}.o"
b._run([b.NVCC, *b.NVFLAGS, "-c", str(b.CSRC / "vxm_unity.cu"), "-o", o])
b._run([b.NVCC, *b.ARCH, "-shared", o, "-o", f"{root}/paper_2112_13169_b200/lib/libvxm_{tag}.so"])
PY
)
git worktree remove --force "$wt"
echo "built paper_2112_13169_b200/lib/libvxm_$tag.so from $rev"
