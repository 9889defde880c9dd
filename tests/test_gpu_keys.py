"""Measurement-key formats (vxm_device.cuh KeyFmt): 16-bit keys (bf16-ordered,
packed-bf16 max reductions) for bundles of up to 32,638 rays, 32-bit keys
above that, with no cap below 2^31 rays (the reference has none,
proj/src/raytracer.cpp:35-61,98-118). Results are identical whichever format
runs, and the keys are left all-Unknown after every merge (so nothing of one
frame leaks into the next: checked by long runs with shifts along every
axis and jumps past the grid)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2112_13169_b200 import _native as N
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests.oracle_api import oracle_pipeline

pytestmark = pytest.mark.gpu
DEG = math.pi / 180.0
KEYS = ("points_total", "points_outside", "rays_traced", "voxels_freed", "voxels_marked_unknown_traced",
        "voxels_skipped_out_of_bounds", "occupied_count", "freed_count", "shifted", "shift_offset", "origin")


def _check(sg, sr, where):
    for key in KEYS:
        assert sg[key] == sr[key], (where, key, sg[key], sr[key])


def test_large_bundle_beyond_the_old_17_bit_ray_cap(gpu_lib):
    """0.03 m voxels at 6.5 m: 217 x 403 x 535 -> 215,605 rays (the previous
    key format capped bundles at 131,070). 32-bit keys; vs the reference."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)
    grid = vm.GridSpec.create_centered(4.5, 4.5, 2.4, 0.03, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    vd, vw, vh = vm.bundle_dimensions(cam, 6.5, 0.03)
    assert vw * vh > 131070
    gpu, orc = vm.MappingPipeline(cfg), oracle_pipeline(cfg)
    boxes = scenes.box_field_boxes(2)
    for k in range(3):
        pose = vm.look_along_x((0.0, 0.031 * k, 0.013 * k))
        depth = scenes.render(cam, pose, boxes)
        _check(gpu.integrate_depth(depth, pose), orc.integrate_depth(depth, pose), k)
    assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0])


@pytest.mark.parametrize("shape,vox", [((640, 480), 0.1), ((320, 240), 0.15)])
def test_narrow_and_wide_keys_agree_while_wandering(gpu_lib, shape, vox):
    """The same wandering trajectory (shifts along x, y and z, turns, jumps
    past the grid) through 16-bit and 32-bit keys, single streams and a
    branched batch: identical stats and grids every frame. 640x480 at 0.1 m
    and 6.5 m is cfg1's 19,239-ray bundle, whose keys cover the bf16 zero and
    subnormal patterns (rays ~16,200-16,400)."""
    W, H = shape
    cam = vm.CameraModel(85 * DEG, 101 * DEG, W, H, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 5.0, 3.0, vox, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    narrow = vm.MappingPipeline(cfg)
    wide = vm.MappingPipeline(cfg, flags=N.FLAG_WIDE_KEYS)
    orc = oracle_pipeline(cfg)
    rng = np.random.default_rng(W)
    p = np.zeros(3)
    boxes = scenes.box_field_boxes(5)
    for i in range(24):
        if i % 9 == 8:
            p = p + np.array([0.0, 7.0, 0.0])  # past the grid
        else:
            p = p + rng.uniform(-0.2, 0.2, 3)
        yaw = rng.uniform(-0.25, 0.25)
        R = vm.look_along_x((0, 0, 0))[0] @ np.array([[math.cos(yaw), 0, math.sin(yaw)], [0, 1, 0],
                                                      [-math.sin(yaw), 0, math.cos(yaw)]])
        pose = (R, p.copy())
        depth = scenes.render(cam, pose, boxes)
        sn, sw = narrow.integrate_depth(depth, pose), wide.integrate_depth(depth, pose)
        sr = orc.integrate_depth(depth, pose)
        _check(sn, sr, ("narrow", i))
        _check(sw, sr, ("wide", i))
        if i % 6 == 5:
            rc = orc.local_grid()[0]
            assert np.array_equal(narrow.local_grid()[0], rc), i
            assert np.array_equal(wide.local_grid()[0], rc), i
