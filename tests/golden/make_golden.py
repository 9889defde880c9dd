"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE's own
code (oracle/_ref/libvoxmap_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile.ref). Run in the build container, where /root/reference
exists:

    python tests/golden/make_golden.py

Outputs (committed):
  box_field_scenes.json   Scene::box_field(seed) boxes for seeds 1..8, 109
  golden_vectors.npz      inputs + reference outputs: transform_voxelize,
                          merge, populate (vox_inf 0..3), trace_bundle,
                          shift, depth_to_cloud, and two short pipeline
                          sequences (bundled / per-pixel tracer)
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_2112_13169_b200 import _native as N  # noqa: E402
from paper_2112_13169_b200.voxmap import look_along_x  # noqa: E402

DEG = math.pi / 180.0


def rot(rng):
    axis = rng.uniform(-1, 1, 3)
    axis /= np.linalg.norm(axis)
    ang = rng.uniform(-1, 1) * math.pi
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * (K @ K)


def grid_c(dims, vs, origin=(0.0, 0.0, 0.0)):
    g = N.GridSpecC()
    for a in range(3):
        g.size[a] = dims[a] * vs
        g.dims[a] = dims[a]
        g.origin[a] = origin[a]
    g.vox_size = vs
    return g


def cam_c(w, h, depth):
    return N.CameraC(85 * DEG, 101 * DEG, w, h, depth)


def main():
    scenes = {str(s): ref.box_field(s).tolist() for s in list(range(1, 9)) + [109]}
    (HERE / "box_field_scenes.json").write_text(json.dumps(scenes, indent=0))

    rng = np.random.default_rng(2112)
    out = {}
    # transform_voxelize (kernels.hpp TransformVoxelizeFn), scalar table
    n = 257
    xs, ys, zs = (rng.uniform(-30, 30, n) for _ in range(3))
    xs[:4] = [0.05, 0.15, -0.05, 1e12]
    R, t = rot(rng), rng.uniform(-3, 3, 3)
    out["tv_in"] = np.stack([xs, ys, zs])
    out["tv_R"], out["tv_t"], out["tv_vs"] = R, t, np.array(0.1)
    out["tv_out"] = np.stack(ref.transform_voxelize(xs, ys, zs, R, t, 0.1))
    # merge, all 16 state pairs plus random
    loc = np.concatenate([np.repeat(np.arange(4, dtype=np.uint8), 4), rng.integers(0, 4, 1000, dtype=np.uint8)])
    ms = np.concatenate([np.tile(np.arange(4, dtype=np.uint8), 4), rng.integers(0, 4, 1000, dtype=np.uint8)])
    merged = loc.copy()
    ref.merge(merged, ms)
    out["merge_loc"], out["merge_ms"], out["merge_out"] = loc, ms, merged
    # populate, vox_inf 0..3 (acceptance criterion 4 shape)
    g = grid_c((32, 32, 32), 0.15)
    for r in range(4):
        m = 3000
        p = np.stack([rng.uniform(-0.6, 32 * 0.15 + 0.6, m) for _ in range(3)])
        pose = (rot(rng), rng.uniform(-0.5, 0.5, 3))
        cells = np.zeros(32 ** 3, dtype=np.uint8)
        st = ref.populate(g, cells, p[0], p[1], p[2], pose, r)
        out[f"pop{r}_pts"], out[f"pop{r}_R"], out[f"pop{r}_t"] = p, pose[0], pose[1]
        out[f"pop{r}_cells"] = cells
        out[f"pop{r}_stats"] = np.array([st["points_total"], st["points_outside"]], dtype=np.uint64)
    # trace_bundle (acceptance criterion 3 shape)
    for k in range(3):
        cells = np.zeros(32 ** 3, dtype=np.uint8)
        idx = rng.integers(0, 32 ** 3, 300)
        cells[idx] = 2
        pose = (rot(rng), rng.uniform(1.2, 3.6, 3))
        before = cells.copy()
        st = ref.trace_bundle(g, cells, (16, 13, 13), pose)
        out[f"tr{k}_in"], out[f"tr{k}_out"] = before, cells
        out[f"tr{k}_R"], out[f"tr{k}_t"] = pose
        out[f"tr{k}_stats"] = np.array([st[k2] for k2, _ in N.TraceStatsC._fields_], dtype=np.uint64)
    # shift
    g2 = grid_c((16, 14, 9), 0.15)
    cells = rng.integers(0, 4, 16 * 14 * 9, dtype=np.uint8)
    offs = np.array([[0, 0, 0], [3, -2, 1], [-5, 4, -3], [20, 0, 0], [-1, -1, -1]], dtype=np.int32)
    out["shift_in"], out["shift_offs"] = cells, offs
    out["shift_out"] = np.stack([ref.shift(g2, cells, o) for o in offs])
    # depth_to_cloud
    cam = cam_c(97, 61, 5.0)
    d = rng.uniform(0.3, 5.2, (61, 97)).astype(np.float32)
    d[rng.random((61, 97)) < 0.05] = 0.0
    d[0, :3] = [np.nan, np.inf, -1.0]
    out["d2c_depth"] = d
    out["d2c_cloud"] = np.stack(ref.depth_to_cloud(cam, d))
    # pipelines: 160x120, 6x6x3 m @ 0.15, vox_inf 1, 6 frames of box_field(1), moving
    cam = cam_c(160, 120, 6.5)
    for mode in (0, 1):
        gc = N.GridSpecC()
        ref._check(ref.lib().ref_grid_spec_create_centered(6.0, 6.0, 3.0, 0.15,
                                                           np.zeros(3).ctypes.data_as(ref._f64p), gc))
        cfg = N.ConfigC(gc, cam, 1, mode, 4.0)
        pipe = ref.Pipeline(cfg)
        stats, frames, poses = [], [], []
        for k in range(6):
            pose = look_along_x((0.03 * k, -0.2 + 0.13 * k, 0.01 * k))
            depth = ref.render_depth(cam, pose, "boxes", seed=1)
            s = pipe.integrate_depth(depth, pose)
            frames.append(depth)
            poses.append(np.concatenate([np.asarray(pose[0]).ravel(), pose[1]]))
            stats.append([s[k2] for k2 in ("points_total", "points_outside", "rays_traced", "voxels_freed",
                                           "voxels_marked_unknown_traced", "voxels_skipped_out_of_bounds",
                                           "occupied_count", "freed_count", "shifted")])
        cells, origin = pipe.local_grid()
        tag = "pipe_bundled" if mode == 0 else "pipe_perpixel"
        out[f"{tag}_depth"] = np.stack(frames)
        out[f"{tag}_poses"] = np.stack(poses)
        out[f"{tag}_stats"] = np.array(stats, dtype=np.uint64)
        out[f"{tag}_cells"] = cells
        out[f"{tag}_origin"] = origin
    np.savez_compressed(HERE / "golden_vectors.npz", **out)
    print("wrote", HERE / "golden_vectors.npz", (HERE / "golden_vectors.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
