"""Randomised parity sweep of the stand-alone stage entry points (test
infrastructure; run under gpurun): populate_occupied (random clouds, poses,
vox_inf 0-6, pre-existing states), trace_bundle (random bundles, cameras inside
and outside the grid, random occupancy and pre-existing states), shift_grid_by
and merge, on random grid shapes, against the reference build.
Usage: python tools/fuzz_stages.py [seconds] [seed]"""
import math, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2112_13169_b200 import voxmap as vm
from oracle import ref


def rot(rng):
    a = rng.uniform(-1, 1, 3)
    a /= max(np.linalg.norm(a), 1e-9)
    t = rng.uniform(-math.pi, math.pi)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(t) * K + (1 - math.cos(t)) * (K @ K)


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else int(time.time()) % 100000
    rng = np.random.default_rng(seed)
    print("seed", seed, flush=True)
    t_end = time.time() + budget
    counts = {"populate": 0, "trace": 0, "shift": 0, "merge": 0}
    while time.time() < t_end:
        vox = float(rng.choice([0.07, 0.1, 0.15]))
        dims = rng.integers([3, 3, 3], [140, 60, 40])
        grid = vm.GridSpec.create(*(d * vox for d in dims), vox)
        n = grid.cell_count()
        pre = rng.integers(0, 4, n).astype(np.uint8) if rng.random() < 0.5 else np.zeros(n, np.uint8)
        kind = rng.choice(["populate", "trace", "shift", "merge"])
        if kind == "populate":
            m = int(rng.integers(0, 4000))
            ext = np.array(grid.dims) * vox
            xs, ys, zs = (rng.uniform(-0.5, e + 0.5, m) for e in ext)
            pose = (rot(rng), rng.uniform(-0.5, 0.5, 3))
            r = int(rng.integers(0, 7))
            a, b = pre.copy(), pre.copy()
            sr = ref.populate(grid.c, a, xs, ys, zs, pose, r)
            sg = vm.populate_occupied(grid, b, xs, ys, zs, pose, r)
            ok = sr == sg and np.array_equal(a, b)
        elif kind == "trace":
            ms = pre.copy()
            ms[rng.random(n) < rng.uniform(0, 0.05)] = 2
            ext = np.array(grid.dims) * vox
            inside = rng.random() < 0.7
            pos = rng.uniform(0.2, 0.8, 3) * ext if inside else rng.uniform(-0.5, 1.5, 3) * ext
            pose = (rot(rng), pos)
            bundle = (int(rng.integers(1, 40)), 2 * int(rng.integers(0, 15)) + 1, 2 * int(rng.integers(0, 15)) + 1)
            a, b = ms.copy(), ms.copy()
            sr = ref.trace_bundle(grid.c, a, bundle, pose)
            sg = vm.trace_bundle(grid, b, bundle, pose)
            ok = sr == sg and np.array_equal(a, b)
        elif kind == "shift":
            off = tuple(int(v) for v in rng.integers(-dims, dims + 1))
            ok = np.array_equal(vm.shift_grid_by(grid.dims, pre, off), ref.shift(grid.c, pre, off))
        else:
            ms = rng.integers(0, 4, n).astype(np.uint8)
            a, b = pre.copy(), pre.copy()
            ref.merge(a, ms.copy())
            vm.merge_grids(b, ms.copy())
            ok = np.array_equal(a, b)
        if not ok:
            print("MISMATCH", kind, "dims", tuple(grid.dims), "vox", vox, flush=True)
            sys.exit(1)
        counts[kind] += 1
    print("fuzz stages:", counts, "all bit-exact", flush=True)


if __name__ == "__main__":
    main()
