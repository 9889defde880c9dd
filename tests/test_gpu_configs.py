"""Parity at the BASELINE.json configurations:
cfg3 (1280x720, 0.05 m, 200x200x100, full frustum ray casting) and cfg4
(a 1000-frame moving trajectory exercising shift/merge every frame), against
the reference's own Sequential pipeline. Frames come from the reference's
renderer when the build is present (fast, OpenMP), else tests/scenes.py."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests.oracle_api import oracle_pipeline

pytestmark = pytest.mark.gpu
DEG = math.pi / 180.0
KEYS = ("points_total", "points_outside", "rays_traced", "voxels_freed", "voxels_marked_unknown_traced",
        "voxels_skipped_out_of_bounds", "occupied_count", "freed_count", "shifted", "shift_offset", "origin")


def render(cam, pose, boxes):
    try:
        from oracle import ref
        if ref.available():
            return ref.render_depth(cam.to_c(), pose, boxes=boxes)
    except Exception:
        pass
    return scenes.render(cam, pose, boxes)


@pytest.mark.parametrize("vox_inf", [0, 2])
def test_cfg3_1280x720_full_frustum(gpu_lib, vox_inf):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 1280, 720, 6.5)
    grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.05, (0.0, 0.0, 0.0))
    assert grid.dims == (200, 200, 100)
    cfg = vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=6.5)
    assert vm.bundle_dimensions(cam, 6.5, 0.05) == (130, 239, 317)  # 75,763 rays
    gpu, orc = vm.MappingPipeline(cfg), oracle_pipeline(cfg)
    boxes = scenes.box_field_boxes(3)
    for k in range(2):
        pose = vm.look_along_x((0.0, 0.04 * k, 0.01 * k))
        depth = render(cam, pose, boxes)
        sg, sr = gpu.integrate_depth(depth, pose), orc.integrate_depth(depth, pose)
        for key in KEYS:
            assert sg[key] == sr[key], (k, key, sg[key], sr[key])
        assert sg["rays_traced"] == 75763
        assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0]), k


def test_cfg4_1000_frame_trajectory(gpu_lib):
    """sweep_trajectory((0,-50,0),(0,50,0),1000): 0.1001 m per
    frame, about one y-shift per frame, cfg1 grid, corridor scene."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)  # reduced image: the oracle runs 1000 frames
    grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0.0, -50.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=0, depth=6.5)
    gpu, orc = vm.MappingPipeline(cfg), oracle_pipeline(cfg)
    boxes = scenes.corridor_boxes(-60.0, 60.0)
    shifts = 0
    for i in range(1000):
        y = -50.0 + (i / 999) * 100.0
        pose = vm.look_along_x((0.0, y, 0.0))
        depth = render(cam, pose, boxes)
        sg, sr = gpu.integrate_depth(depth, pose), orc.integrate_depth(depth, pose)
        shifts += sr["shifted"]
        for key in KEYS:
            assert sg[key] == sr[key], (i, key, sg[key], sr[key])
        if i % 100 == 99:
            assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0]), i
    assert shifts > 500  # recentring on most frames (the reference's own count is what matters)
