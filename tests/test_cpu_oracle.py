"""Pins the plain-C restatement oracle (oracle/voxmap_oracle.c): byte-exact
against the committed golden vectors (made from the reference's own code by
tests/golden/make_golden.py) and, when the reference build is present,
against oracle/_ref on fresh random cases. CPU only."""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import c_oracle as co
from paper_2112_13169_b200 import _native as N
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests.oracle_api import have_ref

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "golden_vectors.npz")
DEG = math.pi / 180.0


def grid_c(dims, vs, origin=(0.0, 0.0, 0.0)):
    g = N.GridSpecC()
    for a in range(3):
        g.size[a] = dims[a] * vs
        g.dims[a] = dims[a]
        g.origin[a] = origin[a]
    g.vox_size = vs
    return g


def test_golden_transform_voxelize():
    p = GOLD["tv_in"]
    got = co.transform_voxelize(p[0], p[1], p[2], GOLD["tv_R"], GOLD["tv_t"], float(GOLD["tv_vs"]))
    assert np.array_equal(np.stack(got), GOLD["tv_out"])


def test_golden_merge():
    loc = GOLD["merge_loc"].copy()
    co.merge(loc, GOLD["merge_ms"])
    assert np.array_equal(loc, GOLD["merge_out"])


@pytest.mark.parametrize("r", [0, 1, 2, 3])
def test_golden_populate(r):
    g = grid_c((32, 32, 32), 0.15)
    cells = np.zeros(32 ** 3, dtype=np.uint8)
    p = GOLD[f"pop{r}_pts"]
    st = co.populate(g, cells, p[0], p[1], p[2], (GOLD[f"pop{r}_R"], GOLD[f"pop{r}_t"]), r)
    assert [st["points_total"], st["points_outside"]] == list(GOLD[f"pop{r}_stats"])
    assert np.array_equal(cells, GOLD[f"pop{r}_cells"])


@pytest.mark.parametrize("k", [0, 1, 2])
def test_golden_trace_bundle(k):
    g = grid_c((32, 32, 32), 0.15)
    cells = GOLD[f"tr{k}_in"].copy()
    st = co.trace_bundle(g, cells, (16, 13, 13), (GOLD[f"tr{k}_R"], GOLD[f"tr{k}_t"]))
    assert [st[f] for f, _ in N.TraceStatsC._fields_] == list(GOLD[f"tr{k}_stats"])
    assert np.array_equal(cells, GOLD[f"tr{k}_out"])


def test_golden_shift():
    g = grid_c((16, 14, 9), 0.15)
    for off, want in zip(GOLD["shift_offs"], GOLD["shift_out"]):
        assert np.array_equal(co.shift(g, GOLD["shift_in"], off), want)


def test_golden_depth_to_cloud():
    cam = N.CameraC(85 * DEG, 101 * DEG, 97, 61, 5.0)
    got = co.depth_to_cloud(cam, GOLD["d2c_depth"])
    assert np.array_equal(np.stack(got), GOLD["d2c_cloud"])


@pytest.mark.parametrize("tag,mode", [("pipe_bundled", 0), ("pipe_perpixel", 1)])
def test_golden_pipeline_sequences(tag, mode):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=4.0, tracer_mode=mode)
    pipe = co.Pipeline(cfg.to_c())
    for k in range(GOLD[f"{tag}_depth"].shape[0]):
        pv = GOLD[f"{tag}_poses"][k]
        s = pipe.integrate_depth(GOLD[f"{tag}_depth"][k], (pv[:9].reshape(3, 3), pv[9:]))
        got = [s[f] for f in ("points_total", "points_outside", "rays_traced", "voxels_freed",
                              "voxels_marked_unknown_traced", "voxels_skipped_out_of_bounds",
                              "occupied_count", "freed_count", "shifted")]
        assert got == list(GOLD[f"{tag}_stats"][k]), k
    cells, origin = pipe.local_grid()
    assert np.array_equal(cells, GOLD[f"{tag}_cells"])
    assert np.array_equal(origin, GOLD[f"{tag}_origin"])


def test_bundle_dimensions_known_answers():
    # proj/tests/test_raytracer.cpp:35-45 and SURVEY Appendix A
    assert co.bundle_dimensions(N.CameraC(85 * DEG, 101 * DEG, 320, 240, 6.5), 6.5, 0.15) == (43, 79, 105)
    assert co.bundle_dimensions(N.CameraC(85 * DEG, 101 * DEG, 640, 480, 5.0), 5.0, 0.1) == (50, 93, 123)


def test_scene_generator_matches_golden_frames():
    # the pipeline golden frames were rendered by the reference's render_depth
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)
    for k in range(GOLD["pipe_bundled_depth"].shape[0]):
        pv = GOLD["pipe_bundled_poses"][k]
        got = scenes.render(cam, (pv[:9].reshape(3, 3), pv[9:]), scenes.box_field_boxes(1))
        assert np.array_equal(got, GOLD["pipe_bundled_depth"][k])


# ---------------------------------------------------------------- vs the reference build

needs_ref = pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")


def _rot(rng):
    axis = rng.uniform(-1, 1, 3)
    axis /= np.linalg.norm(axis)
    ang = rng.uniform(-1, 1) * math.pi
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * (K @ K)


@needs_ref
def test_oracle_equals_reference_random_stages():
    from oracle import ref

    rng = np.random.default_rng(77)
    g = grid_c((24, 20, 16), 0.15, (0.1, -0.2, 0.05))
    for _ in range(20):
        pose = (_rot(rng), rng.uniform(0.5, 2.5, 3))
        n = int(rng.integers(0, 2000))
        p = [rng.uniform(-1, 4, n) for _ in range(3)]
        r = int(rng.integers(0, 4))
        a = np.zeros(24 * 20 * 16, dtype=np.uint8)
        b = a.copy()
        assert co.populate(g, a, *p, pose, r) == ref.populate(g, b, *p, pose, r)
        assert np.array_equal(a, b)
        bundle = (int(rng.integers(5, 20)), 2 * int(rng.integers(1, 9)) + 1, 2 * int(rng.integers(1, 9)) + 1)
        assert co.trace_bundle(g, a, bundle, pose) == ref.trace_bundle(g, b, bundle, pose)
        assert np.array_equal(a, b)
        c1, c2 = a.copy(), b.copy()
        assert co.trace_per_pixel(g, c1, *p, pose) == ref.trace_per_pixel(g, c2, *p, pose)
        assert np.array_equal(c1, c2)


@needs_ref
@pytest.mark.parametrize("mode", [0, 1])
def test_oracle_equals_reference_pipeline(mode):
    from oracle import ref

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 128, 96, 6.5)
    grid = vm.GridSpec.create_centered(8.0, 8.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0, tracer_mode=mode)
    a, b = co.Pipeline(cfg.to_c()), ref.Pipeline(cfg.to_c())
    for k in range(12):
        pose = vm.look_along_x((0.02 * k, -0.5 + 0.12 * k, 0.0))
        depth = scenes.render(cam, pose, scenes.box_field_boxes(2))
        sa, sb = a.integrate_depth(depth, pose), b.integrate_depth(depth, pose)
        for key in ("points_total", "rays_traced", "voxels_freed", "voxels_marked_unknown_traced",
                    "occupied_count", "freed_count", "shifted", "shift_offset", "origin"):
            assert sa[key] == sb[key], (k, key)
        assert np.array_equal(a.local_grid()[0], b.local_grid()[0])
