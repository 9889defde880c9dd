"""Multi-frame pipelining (SURVEY.md §8f "next" #1): F consecutive frames of
each stream per call (vxm_create_multi). Every frame's stats and the local
grid after each call must equal F successive single-frame integrations —
against the reference's Sequential build (oracle/_ref) and against the
single-frame GPU path — bit for bit, including shifts along every axis,
back-and-forth motion and jumps larger than the grid."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests.oracle_api import have_ref, oracle_pipeline

pytestmark = pytest.mark.gpu

if not have_ref():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

DEG = math.pi / 180.0
KEYS = ("points_total", "points_outside", "rays_traced", "voxels_freed", "voxels_marked_unknown_traced",
        "voxels_skipped_out_of_bounds", "occupied_count", "freed_count", "shifted", "shift_offset", "origin")


def _check(sg, sr, where):
    for key in KEYS:
        assert sg[key] == sr[key], (where, key, sg[key], sr[key])


def test_sequence_matches_reference_along_a_corridor(gpu_lib):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 64, 48, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, -8.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    boxes = scenes.corridor_boxes(-12.0, 25.0)
    F = 8
    seq = vm.MappingPipeline(cfg, frames_per_call=F)
    orc = oracle_pipeline(cfg)
    k = 0
    for call in range(5):
        poses = [vm.look_along_x((0.0, -8.0 + 0.1001 * (k + j), 0.0)) for j in range(F)]
        depth = np.stack([scenes.render(cam, p, boxes) for p in poses])
        stats = seq.integrate_depth(depth, poses)
        for j in range(F):
            _check(stats[j], orc.integrate_depth(depth[j], poses[j]), (call, j))
        k += F
        cells, origin = seq.local_grid()
        rc, ro = orc.local_grid()
        assert np.array_equal(cells, rc), call
        assert np.array_equal(origin, ro)


def _wander(rng, n, start):
    """Poses that shift along x, y and z, turn back, stand still and jump
    further than the grid is wide."""
    p = np.array(start, dtype=float)
    out = []
    for i in range(n):
        if i % 11 == 7:
            p = p + np.array([0.0, 9.0 if (i // 11) % 2 == 0 else -9.0, 0.0])  # jump past the grid
        elif i % 5 == 3:
            pass  # stand still
        else:
            p = p + rng.uniform(-0.17, 0.17, 3) * np.array([1.0, 1.0, 0.6])
        yaw = rng.uniform(-0.3, 0.3)
        R = vm.look_along_x((0, 0, 0))[0] @ np.array([[math.cos(yaw), 0, math.sin(yaw)], [0, 1, 0],
                                                      [-math.sin(yaw), 0, math.cos(yaw)]])
        out.append((R, p.copy()))
    return out


@pytest.mark.parametrize("S,F", [(1, 3), (2, 7), (3, 16), (5, 4), (1, 33), (1, 64)])
def test_sequence_equals_single_frame_path_while_wandering(gpu_lib, S, F):
    """(1, 33) and (1, 64): a single stream with F >= 32 merges its frame
    ranges as chained per-branch merges (uneven ranges for 33)."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 96, 72, 6.5)
    grid = vm.GridSpec.create_centered(5.0, 4.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=6.0)
    rng = np.random.default_rng(100 * S + F)
    calls = 3
    trajs = [_wander(rng, calls * F, (0.05 * s, 0.0, 0.0)) for s in range(S)]
    boxes = [scenes.box_field_boxes(3 + s) for s in range(S)]
    seq = vm.MappingPipeline(cfg, n_streams=S, frames_per_call=F)
    singles = [vm.MappingPipeline(cfg) for _ in range(S)]
    for call in range(calls):
        poses = [trajs[s][call * F + j] for s in range(S) for j in range(F)]
        depth = np.stack([scenes.render(cam, poses[s * F + j], boxes[s]) for s in range(S) for j in range(F)])
        stats = seq.integrate_depth(depth, poses)
        for s in range(S):
            for j in range(F):
                i = s * F + j
                _check(stats[i], singles[s].integrate_depth(depth[i], poses[i]), (call, s, j))
            assert np.array_equal(seq.local_grid(s)[0], singles[s].local_grid()[0]), (call, s)
            assert np.array_equal(seq.local_grid(s)[1], singles[s].local_grid()[1])
    # and the single-frame path against the reference build on the last stream
    orc = oracle_pipeline(cfg)
    for i in range(calls * F):
        pose = trajs[S - 1][i]
        orc.integrate_depth(scenes.render(cam, pose, boxes[S - 1]), pose)
    assert np.array_equal(seq.local_grid(S - 1)[0], orc.local_grid()[0])


def test_sequence_device_frames_and_restored_grid(gpu_lib):
    """Device-resident frames (the bench path) and a local grid restored from
    a checkpoint before the first call."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 80, 60, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=0, depth=6.5)
    F = 5
    rng = np.random.default_rng(5)
    start = rng.integers(0, 4, grid.cell_count()).astype(np.uint8)
    seq = vm.MappingPipeline(cfg, frames_per_call=F)
    one = vm.MappingPipeline(cfg)
    org = grid.origin + np.array([0.3, -0.15, 0.0])
    seq.set_local_grid(start, org)
    one.set_local_grid(start, org)
    poses = [vm.look_along_x((0.0, 0.13 * j - 0.3, 0.02 * j)) for j in range(F)]
    depth = np.stack([scenes.render(cam, p, scenes.box_field_boxes(2)) for p in poses])
    dev = torch.from_numpy(depth).cuda()
    seq.integrate_depth_device(dev.data_ptr(), poses)
    stats = seq.wait_stats()
    for j in range(F):
        _check(stats[j], one.integrate_depth(depth[j], poses[j]), j)
    assert np.array_equal(seq.local_grid()[0], one.local_grid()[0])


def test_sequence_argument_checks(gpu_lib):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 32, 24, 6.5)
    grid = vm.GridSpec.create_centered(3.0, 3.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=0, depth=6.5)
    for bad in (0, -1, 65):
        with pytest.raises(ValueError, match="frames_per_call"):
            vm.MappingPipeline(cfg, frames_per_call=bad)
    seq = vm.MappingPipeline(cfg, frames_per_call=2)
    with pytest.raises(ValueError):
        seq.integrate_depth(np.ones((24, 32), np.float32), [vm.look_along_x((0, 0, 0))])
    with pytest.raises(ValueError, match="single-frame"):
        seq.integrate(np.ones(3), np.ones(3), np.ones(3), vm.look_along_x((0, 0, 0)))


def test_sequence_partial_calls_host_frames(gpu_lib):
    """vxm_integrate_depth_frames: 1..F host frames per call on a
    single-stream multi-frame context (the C++ integrate_depth_sequence path)."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 80, 60, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 5.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    seq = vm.MappingPipeline(cfg, frames_per_call=8)
    one = vm.MappingPipeline(cfg)
    rng = np.random.default_rng(11)
    traj = _wander(rng, 3 + 8 + 1 + 5 + 8, (0.0, 0.0, 0.0))
    i = 0
    for n in (3, 8, 1, 5, 8):
        poses = traj[i:i + n]
        depth = np.stack([scenes.render(cam, p, scenes.box_field_boxes(4)) for p in poses])
        stats = seq.integrate_depth_frames(depth, poses)
        assert len(stats) == n
        for j in range(n):
            _check(stats[j], one.integrate_depth(depth[j], poses[j]), (n, j))
        assert np.array_equal(seq.local_grid()[0], one.local_grid()[0]), n
        i += n
    with pytest.raises(ValueError, match="n_frames"):
        seq.integrate_depth_frames(np.zeros((9, 60, 80), np.float32), traj[:9])


def test_chained_desync_calls_mixed_with_partial_calls(gpu_lib):
    """F = 40 on one stream: full calls run desynchronised branch streams with
    chained range merges (the next call's populate/trace may start before
    this call's merges end); partial calls in between run on the context
    stream. Every frame's stats and the grid equal the single-frame path."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 64, 48, 6.5)
    grid = vm.GridSpec.create_centered(5.0, 4.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=6.0)
    F = 40
    seq = vm.MappingPipeline(cfg, frames_per_call=F)
    one = vm.MappingPipeline(cfg)
    rng = np.random.default_rng(40)
    plan = [F, F, 7, F, 1, F, F]
    traj = _wander(rng, sum(plan), (0.0, 0.0, 0.0))
    boxes = scenes.box_field_boxes(5)
    i = 0
    for n in plan:
        poses = traj[i:i + n]
        depth = np.stack([scenes.render(cam, p, boxes) for p in poses])
        if n == F:
            # device frames, asynchronous: queue it, check after the next call
            dev = torch.from_numpy(depth).cuda()
            seq.integrate_depth_device(dev.data_ptr(), vm.pose_array(poses))
            stats = seq.wait_stats()
        else:
            stats = seq.integrate_depth_frames(depth, poses)
        for j in range(n):
            _check(stats[j], one.integrate_depth(depth[j], poses[j]), (i, n, j))
        assert np.array_equal(seq.local_grid()[0], one.local_grid()[0]), i
        i += n


@pytest.mark.parametrize("F", [40, 64])
def test_full_frames_call_from_pinned_buffer(gpu_lib, F):
    """vxm_integrate_depth_frames with n_frames == F >= 32 from a pinned host
    buffer: the call runs the desynchronised chained-range branches, which
    must not start populating before the H2D copy of the frames has landed
    (the copy is read asynchronously from pinned memory). Checked against the
    reference build frame by frame, twice in a row."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 320, 240, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    seq = vm.MappingPipeline(cfg, frames_per_call=F)
    orc = oracle_pipeline(cfg)
    rng = np.random.default_rng(F)
    traj = _wander(rng, 2 * F, (0.0, 0.0, 0.0))
    boxes = scenes.box_field_boxes(2)
    for call in range(2):
        poses = traj[call * F:(call + 1) * F]
        depth = vm.render_depth(cam, poses, boxes)
        pinned = torch.from_numpy(depth).pin_memory()
        stats = seq.integrate_depth_frames_ptr(pinned.data_ptr(), poses)
        for j in range(F):
            _check(stats[j], orc.integrate_depth(depth[j], poses[j]), (call, j))
        assert np.array_equal(seq.local_grid()[0], orc.local_grid()[0]), call
