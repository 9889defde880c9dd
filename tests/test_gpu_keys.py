"""Measurement-key formats (vxm_device.cuh KeyFmt): epoch-tagged keys for
bundles of up to 131,070 rays (every BASELINE config), and the clear format
(no epochs; the merge resets every key it reads and the cells the shift drops)
above that, with no cap below 2^31 rays (the reference has none,
proj/src/raytracer.cpp:35-61,98-118). Results are identical whichever format
runs; long runs with shifts along every axis and jumps past the grid check
that nothing of one frame leaks into the next. Also the generic dilation for
radii and rows beyond the tile kernels."""
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
    """0.03 m voxels at 6.5 m: more than 131,070 rays (the epoch format's
    17-bit ray field), so the clear format runs; vs the reference."""
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
def test_epoch_and_clear_keys_agree_while_wandering(gpu_lib, shape, vox):
    """The same wandering trajectory (shifts along x, y and z, turns, jumps
    past the grid) through both key formats (VXM_FLAG_CLEAR_KEYS forces the
    clear format): identical stats and grids every frame, equal to the
    reference."""
    W, H = shape
    cam = vm.CameraModel(85 * DEG, 101 * DEG, W, H, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 5.0, 3.0, vox, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    epoch_k = vm.MappingPipeline(cfg)
    clear_k = vm.MappingPipeline(cfg, flags=N.FLAG_CLEAR_KEYS)
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
        sn, sw = epoch_k.integrate_depth(depth, pose), clear_k.integrate_depth(depth, pose)
        sr = orc.integrate_depth(depth, pose)
        _check(sn, sr, ("epoch_k", i))
        _check(sw, sr, ("clear_k", i))
        if i % 6 == 5:
            rc = orc.local_grid()[0]
            assert np.array_equal(epoch_k.local_grid()[0], rc), i
            assert np.array_equal(clear_k.local_grid()[0], rc), i


@pytest.mark.parametrize("vox_inf,size,vox,shape", [
    (20, (6.0, 6.0, 3.0), 0.1, (32, 24)),      # radius beyond the tile kernels (<= 16)
    (17, (4.0, 4.0, 2.0), 0.05, (24, 18)),
    (2, (55.0, 0.5, 0.4), 0.05, (64, 48)),     # rows of 1100 cells (> 1024)
])
def test_generic_dilation_matches_reference(gpu_lib, vox_inf, size, vox, shape):
    """Obstacle inflation the reference accepts for any vox_inf and grid
    (proj/src/integrator.cpp:62-85): radii and row lengths beyond the tile
    dilation take the generic separable line passes."""
    W, H = shape
    cam = vm.CameraModel(85 * DEG, 101 * DEG, W, H, 6.5)
    grid = vm.GridSpec.create_centered(*size, vox, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=6.5)
    gpu, orc = vm.MappingPipeline(cfg), oracle_pipeline(cfg)
    boxes = scenes.box_field_boxes(3)
    for k in range(3):
        pose = vm.look_along_x((0.0, 0.07 * k, 0.0))
        depth = scenes.render(cam, pose, boxes)
        _check(gpu.integrate_depth(depth, pose), orc.integrate_depth(depth, pose), k)
    assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0])
    # the stage entry point too (populate_occupied on a host grid)
    rng = np.random.default_rng(vox_inf)
    ms = rng.integers(0, 4, grid.cell_count()).astype(np.uint8)
    pts = rng.uniform(-0.5, 0.5, (3, 200)) * np.array([[size[0]], [size[1]], [size[2]]])
    from oracle import ref
    t = vm.identity_pose(tuple(-np.asarray(grid.origin)))
    a = ms.copy()
    sa = vm.populate_occupied(grid, a, pts[0], pts[1], pts[2], t, vox_inf)
    b = ms.copy()
    sb = ref.populate(grid.c, b, pts[0], pts[1], pts[2], t, vox_inf)
    assert sa == sb and np.array_equal(a, b)


@pytest.mark.parametrize("S,F", [(13, 1), (1, 40), (3, 8)])
def test_clear_keys_batched_and_multi_frame(gpu_lib, S, F):
    """The clear format through the batched graphs (desynchronised branches),
    the chain-folded multi-frame merge (keys read along every chain, shifted
    out ones reset too) and the chained-range path, against the epoch format."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 96, 72, 6.5)
    grid = vm.GridSpec.create_centered(5.0, 4.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=6.0)
    a = vm.MappingPipeline(cfg, n_streams=S, frames_per_call=F)
    b = vm.MappingPipeline(cfg, n_streams=S, frames_per_call=F, flags=N.FLAG_CLEAR_KEYS)
    rng = np.random.default_rng(S * 100 + F)
    pos = [np.zeros(3) for _ in range(S)]
    boxes = scenes.box_field_boxes(4)
    for call in range(6):
        poses = []
        for s in range(S):
            for j in range(F):
                pos[s] = pos[s] + (np.array([0, 6.0, 0]) if rng.random() < 0.05 else rng.uniform(-0.17, 0.17, 3))
                poses.append(vm.look_along_x(tuple(pos[s])))
        depth = vm.render_depth(cam, poses, boxes)
        dev = torch.from_numpy(depth).cuda()
        a.integrate_depth_device(dev.data_ptr(), vm.pose_array(poses))
        b.integrate_depth_device(dev.data_ptr(), vm.pose_array(poses))
        sa, sb = a.wait_stats(), b.wait_stats()
        for i in range(S * F):
            _check(sb[i], sa[i], (call, i))
    for s in range(S):
        assert np.array_equal(a.local_grid(s)[0], b.local_grid(s)[0]), s


def test_grid_beyond_2_31_cells(gpu_lib):
    """A local grid of 2048 x 1024 x 1025 = 2,149,580,800 cells (> 2^31; the
    reference accepts any size, proj/src/grid.cpp:17-42): 32-bit cell indices
    in modular arithmetic cover grids of up to 2^32 - 2 cells. Rows of 2048
    cells also take the generic dilation and the row-wise merge. Two frames,
    the second recentring the grid, against the reference (which needs ~6 GB
    of host memory here)."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 64, 48, 3.0)
    grid = vm.GridSpec.create_centered(204.8, 102.4, 102.5, 0.1, (0.0, 0.0, 0.0))
    assert grid.dims == (2048, 1024, 1025) and grid.cell_count() > 2 ** 31
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=3.0)
    gpu, orc = vm.MappingPipeline(cfg), oracle_pipeline(cfg)
    boxes = np.array([[1.5, -2.0, -1.0, 1.8, 2.0, 1.0], [2.2, -0.5, -2.0, 2.5, 0.5, 0.5]])
    for k, pos in enumerate([(0.0, 0.0, 0.0), (0.05, 0.27, -0.13)]):
        pose = vm.look_along_x(pos)
        depth = scenes.render(cam, pose, boxes)
        sg, sr = gpu.integrate_depth(depth, pose), orc.integrate_depth(depth, pose)
        _check(sg, sr, k)
    assert sr["shifted"]
    assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0])
    with pytest.raises(ValueError, match="2\\^32"):
        vm.MappingPipeline(vm.PipelineConfig(vm.GridSpec.create_centered(204.8, 204.8, 102.5, 0.1, (0, 0, 0)),
                                             cam, vox_inf=0, depth=3.0))
