"""Parity of the sm_100a path (through the C-ABI) with the reference's own
Sequential implementation (oracle/_ref, or the C restatement). Bit-exact:
grids byte for byte, every counter equal."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2112_13169_b200 import _native as N
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests.oracle_api import have_ref, oracle_pipeline

pytestmark = pytest.mark.gpu

ref = pytest.importorskip("oracle.ref")
if not have_ref():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

DEG = math.pi / 180.0


def random_rotation(rng):
    axis = rng.uniform(-1, 1, 3)
    while np.linalg.norm(axis) < 1e-3:
        axis = rng.uniform(-1, 1, 3)
    axis = axis / np.linalg.norm(axis)
    ang = rng.uniform(-1, 1) * math.pi
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * (K @ K)


# --- KernelTable adapter (proj/tests/test_kernels.cpp) ------------------------

def test_kernel_isa(gpu_lib):
    assert vm.kernel_isa() == "cuda-sm100a"


def test_merge_table_all_16_cases(gpu_lib):
    # proj/tests/test_kernels.cpp:12-21: m==0 keeps, m==3 -> 0, else m
    loc = np.repeat(np.arange(4, dtype=np.uint8), 4)
    ms = np.tile(np.arange(4, dtype=np.uint8), 4)
    expect = np.where(ms == 0, loc, np.where(ms == 3, 0, ms)).astype(np.uint8)
    got = loc.copy()
    vm.kernel_merge(got, ms)
    assert np.array_equal(got, expect)


@pytest.mark.parametrize("n", [0, 1, 15, 16, 31, 32, 33, 100, 4097])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_merge_matches_reference_any_size_and_alignment(gpu_lib, n, offset):
    rng = np.random.default_rng(n * 7 + offset)
    buf_l = rng.integers(0, 4, n + offset, dtype=np.uint8)
    buf_m = rng.integers(0, 4, n + offset, dtype=np.uint8)
    loc, ms = buf_l[offset:], buf_m[offset:]
    want = loc.copy()
    ref.merge(want, ms.copy())
    vm.kernel_merge(loc, ms)
    assert np.array_equal(loc, want)


def test_stage_calls_reuse_scratch(gpu_lib):
    # stage entry points draw their device buffers from a per-thread cache
    # (no cudaMalloc/cudaFree per call): many calls of varying sizes stay
    # bit-exact and leave the device's free memory where the first call left it
    import torch

    rng = np.random.default_rng(5)
    sizes = [int(x) for x in rng.integers(1, 300_000, 40)]
    vm.kernel_merge(np.zeros(300_000, np.uint8), np.zeros(300_000, np.uint8))
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for n in sizes * 3:
        loc = rng.integers(0, 4, n, dtype=np.uint8)
        ms = rng.integers(0, 4, n, dtype=np.uint8)
        want = loc.copy()
        ref.merge(want, ms.copy())
        vm.kernel_merge(loc, ms)
        assert np.array_equal(loc, want), n
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 << 20, (free0, free1)


def test_transform_voxelize_known_answers(gpu_lib):
    # proj/tests/test_kernels.cpp:63-87: floor semantics and the +-1e9 clamp
    xs = np.array([0.05, 0.15, -0.05, 1e12, -1e12, 0.0])
    ys = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    zs = np.array([0.0, 0.25, 0.0, 0.0, 0.0, -0.0])
    R = np.eye(3)
    t = np.zeros(3)
    got = vm.kernel_transform_voxelize(xs, ys, zs, R, t, 0.1)
    want = ref.transform_voxelize(xs, ys, zs, R, t, 0.1)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    assert list(got[0][:3]) == [0, 1, -1]
    assert got[0][3] == 1_000_000_000 and got[0][4] == -1_000_000_000


def test_transform_voxelize_clamp_band_and_near_integers(gpu_lib):
    # quotients just inside / outside the +-1e9 clamp (kernels_scalar.cpp:31-34),
    # around 2^29..2^31, exact multiples of the voxel size, tiny and negative
    # values, NaN and inf: the division-free fast path must agree everywhere
    vs = 0.1
    q = np.array([1e9 - 1.5, 1e9 - 0.5, 1e9, 1e9 + 0.5, 1.05e9, 2.0**29 - 0.5, 2.0**29 + 0.5,
                  2.0**30, 2.0**31 + 7, -1e9 + 0.5, -1e9 - 0.5, -1.05e9, -(2.0**29) - 0.5])
    xs = np.concatenate([q * vs, np.arange(-50, 51) * vs, np.arange(-50, 51) * vs + 1e-17,
                         [1e-300, -1e-300, 5e-324, -0.0, np.nan, np.inf, -np.inf]])
    rng = np.random.default_rng(7)
    xs = np.concatenate([xs, rng.integers(-10**6, 10**6, 2000) * vs,
                         rng.integers(-10**6, 10**6, 2000) * vs * (1 + 1e-15)])
    ys = rng.uniform(-1, 1, xs.size) * 0.0
    zs = np.zeros(xs.size)
    R = np.eye(3)
    t = np.zeros(3)
    got = vm.kernel_transform_voxelize(xs, ys, zs, R, t, vs)
    want = ref.transform_voxelize(xs, ys, zs, R, t, vs)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("vs", [0.05, 0.07, 0.1, 0.15, 0.2, 0.3])
def test_transform_voxelize_near_integer_quotients(gpu_lib, vs):
    """Coordinates within a few ulps of whole multiples of the voxel size and
    of the points where acc / vs rounds across an integer (k - ulp/2): the
    near-integer floor (remainder sign, no division) against the reference's
    floor(acc / vs), positive and negative, up to 2^28 cells."""
    rng = np.random.default_rng(int(vs * 1000))
    k = np.concatenate([np.arange(-40, 41), rng.integers(-2**28, 2**28, 300),
                        2.0 ** np.arange(1, 29), -(2.0 ** np.arange(1, 29))]).astype(np.float64)
    below = np.nextafter(k, -np.inf)
    bases = [k * vs, ((k + below) / 2) * vs]  # multiples, and the rounding midpoints below k
    xs = []
    for b in bases:
        for j in range(-6, 7):
            v = b.copy()
            step = np.inf if j > 0 else -np.inf
            for _ in range(abs(j)):
                v = np.nextafter(v, step)
            xs.append(v)
    xs = np.concatenate(xs)
    zs = np.zeros(xs.size)
    for t0 in (0.0, 0.25, -3.5):
        t = np.array([t0, 0.0, 0.0])
        got = vm.kernel_transform_voxelize(xs, zs, zs, np.eye(3), t, vs)
        want = ref.transform_voxelize(xs, zs, zs, np.eye(3), t, vs)
        for g, w in zip(got, want):
            assert np.array_equal(g, w), (vs, t0, int((g != w).sum()))


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 33, 4097])
def test_transform_voxelize_random_rotations(gpu_lib, n):
    rng = np.random.default_rng(41 + n)
    for _ in range(5):
        xs, ys, zs = (rng.uniform(-20, 20, n) for _ in range(3))
        R = random_rotation(rng)
        t = rng.uniform(-5, 5, 3)
        vs = float(rng.choice([0.05, 0.1, 0.15, 0.3]))
        got = vm.kernel_transform_voxelize(xs, ys, zs, R, t, vs)
        want = ref.transform_voxelize(xs, ys, zs, R, t, vs)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


# --- populate_occupied (proj/tests/test_integrator.cpp, acceptance criterion 4) --

@pytest.mark.parametrize("vox_inf", [0, 1, 2, 3, 4, 5, 8])
def test_populate_matches_reference(gpu_lib, vox_inf):
    rng = np.random.default_rng(104 + vox_inf)
    vox = 0.15
    grid = vm.GridSpec.create(32 * vox, 32 * vox, 32 * vox, vox)
    for n in (1, 500, 5000, 20000):
        xs, ys, zs = (rng.uniform(-0.6, 32 * vox + 0.6, n) for _ in range(3))
        pose = (random_rotation(rng), rng.uniform(-0.5, 0.5, 3))
        ms_ref = np.zeros(grid.cell_count(), dtype=np.uint8)
        ms_gpu = ms_ref.copy()
        st_ref = ref.populate(grid.c, ms_ref, xs, ys, zs, pose, vox_inf)
        st_gpu = vm.populate_occupied(grid, ms_gpu, xs, ys, zs, pose, vox_inf)
        assert st_gpu == st_ref
        assert np.array_equal(ms_gpu, ms_ref)


@pytest.mark.parametrize("dims", [(100, 20, 10), (200, 8, 6), (20, 30, 12), (36, 10, 9), (33, 12, 7),
                                  (64, 5, 5), (96, 7, 3), (8, 9, 10), (4, 4, 4)])
@pytest.mark.parametrize("vox_inf", [1, 2, 5])
def test_populate_dilation_row_layouts(gpu_lib, dims, vox_inf):
    # row lengths that take the vector row-packing path (G*dx a multiple of 16,
    # 1..8 words per row) and ones that fall back to the per-row kernel
    rng = np.random.default_rng(sum(dims) + vox_inf)
    vox = 0.1
    grid = vm.GridSpec.create(dims[0] * vox, dims[1] * vox, dims[2] * vox, vox)
    assert tuple(grid.dims) == dims
    for n in (1, 50, 3000):
        xs, ys, zs = (rng.uniform(-0.3, d * vox + 0.3, n) for d in dims)
        pose = vm.identity_pose()
        # pre-existing states (populate never clears, test_integrator.cpp:127-137)
        ms_ref = rng.integers(0, 4, grid.cell_count()).astype(np.uint8) if n == 50 else \
            np.zeros(grid.cell_count(), dtype=np.uint8)
        ms_gpu = ms_ref.copy()
        st_ref = ref.populate(grid.c, ms_ref, xs, ys, zs, pose, vox_inf)
        st_gpu = vm.populate_occupied(grid, ms_gpu, xs, ys, zs, pose, vox_inf)
        assert st_gpu == st_ref
        assert np.array_equal(ms_gpu, ms_ref)


def test_populate_never_clears_and_is_idempotent(gpu_lib):
    # test_integrator.cpp:107-137
    grid = vm.GridSpec.create(1.5, 1.5, 1.5, 0.15)
    ms = np.zeros(grid.cell_count(), dtype=np.uint8)
    ms[::7] = 1
    ms[::11] = 3
    before = ms.copy()
    xs, ys, zs = np.array([0.7]), np.array([0.7]), np.array([0.7])
    vm.populate_occupied(grid, ms, xs, ys, zs, vm.identity_pose(), 2)
    again = ms.copy()
    vm.populate_occupied(grid, again, xs, ys, zs, vm.identity_pose(), 2)
    assert np.array_equal(ms, again)
    untouched = ms != 2
    assert np.array_equal(ms[untouched], before[untouched])
    assert int((ms == 2).sum()) == 125


# --- trace_bundle (acceptance criterion 3, test_raytracer.cpp) ------------------

def _random_occupied(rng, grid, count):
    ms = np.zeros(grid.cell_count(), dtype=np.uint8)
    d = grid.dims
    for _ in range(count):
        x, y, z = rng.integers(0, d[0]), rng.integers(0, d[1]), rng.integers(0, d[2])
        ms[x + y * d[0] + z * d[0] * d[1]] = 2
    return ms


def test_trace_bundle_matches_sequential_reference(gpu_lib):
    vox = 0.15
    grid = vm.GridSpec.create(32 * vox, 32 * vox, 32 * vox, vox)
    rng = np.random.default_rng(103)
    for scene in range(40):
        ms = _random_occupied(rng, grid, int(rng.integers(50, 400)))
        pose = (random_rotation(rng), rng.uniform(1.2, 3.6, 3))
        bundle = (16, 13, 13)
        ms_ref, ms_gpu = ms.copy(), ms.copy()
        st_ref = ref.trace_bundle(grid.c, ms_ref, bundle, pose)
        st_gpu = vm.trace_bundle(grid, ms_gpu, bundle, pose)
        assert st_gpu == st_ref, scene
        assert np.array_equal(ms_gpu, ms_ref), (scene, int((ms_gpu != ms_ref).sum()))


def test_trace_bundle_camera_outside_grid_counts_skips(gpu_lib):
    vox = 0.15
    grid = vm.GridSpec.create(24 * vox, 24 * vox, 24 * vox, vox)
    rng = np.random.default_rng(7)
    for k in range(10):
        ms = _random_occupied(rng, grid, 200)
        pose = vm.look_along_x((-1.0 - 0.1 * k, 1.8, 1.8))
        ms_ref, ms_gpu = ms.copy(), ms.copy()
        st_ref = ref.trace_bundle(grid.c, ms_ref, (40, 31, 31), pose)
        st_gpu = vm.trace_bundle(grid, ms_gpu, (40, 31, 31), pose)
        assert st_ref["voxels_skipped_out_of_bounds"] > 0
        assert st_gpu == st_ref
        assert np.array_equal(ms_gpu, ms_ref)


def test_trace_bundle_preexisting_free_and_traced(gpu_lib):
    vox = 0.15
    grid = vm.GridSpec.create(20 * vox, 20 * vox, 20 * vox, vox)
    rng = np.random.default_rng(11)
    ms = rng.integers(0, 4, grid.cell_count(), dtype=np.uint8)
    pose = vm.look_along_x((0.3, 1.5, 1.5))
    ms_ref, ms_gpu = ms.copy(), ms.copy()
    assert vm.trace_bundle(grid, ms_gpu, (15, 11, 11), pose) == ref.trace_bundle(grid.c, ms_ref, (15, 11, 11), pose)
    assert np.array_equal(ms_gpu, ms_ref)


def test_trace_bundle_rejects_bad_bundle(gpu_lib):
    grid = vm.GridSpec.create(1.5, 1.5, 1.5, 0.15)
    ms = np.zeros(grid.cell_count(), dtype=np.uint8)
    with pytest.raises(ValueError):
        vm.trace_bundle(grid, ms, (10, 4, 5), vm.identity_pose())


# --- shift and depth_to_cloud ----------------------------------------------------

def test_shift_matches_reference(gpu_lib):
    grid = vm.GridSpec.create(16 * 0.15, 14 * 0.15, 9 * 0.15, 0.15)
    rng = np.random.default_rng(111)
    for _ in range(50):
        cells = rng.integers(0, 4, grid.cell_count(), dtype=np.uint8)
        off = rng.integers(-20, 21, 3) if rng.random() < 0.3 else rng.integers(-5, 6, 3)
        assert np.array_equal(vm.shift_grid_by(grid.dims, cells, off), ref.shift(grid.c, cells, off))


def test_depth_to_cloud_matches_reference(gpu_lib):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 97, 61, 5.0)
    depth = scenes.stress_depth(cam, seed=3)
    depth[0, :5] = [np.nan, np.inf, -1.0, 5.0, 5.0000005]
    got = vm.depth_to_cloud(depth, cam)
    want = ref.depth_to_cloud(cam.to_c(), depth)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


# --- the full per-frame pipeline ------------------------------------------------

def _run_pair(cfg, frames):
    gpu = vm.MappingPipeline(cfg)
    orc = oracle_pipeline(cfg)
    for k, (depth, pose) in enumerate(frames):
        sg = gpu.integrate_depth(depth, pose)
        sr = orc.integrate_depth(depth, pose)
        for key in ("points_total", "points_outside", "rays_traced", "voxels_freed",
                    "voxels_marked_unknown_traced", "voxels_skipped_out_of_bounds", "occupied_count",
                    "freed_count", "shifted", "shift_offset", "origin"):
            assert sg[key] == sr[key], (k, key, sg[key], sr[key])
        cg, og = gpu.local_grid()
        cr, orr = orc.local_grid()
        assert np.array_equal(og, orr)
        assert np.array_equal(cg, cr), (k, int((cg != cr).sum()))
    return gpu


@pytest.mark.parametrize("vox_inf", [0, 2])
def test_pipeline_reference_default_config_moving(gpu_lib, vox_inf):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 320, 240, 6.5)
    grid = vm.GridSpec.create_centered(15.0, 15.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=6.5)
    boxes = scenes.box_field_boxes(1)
    frames = []
    for k in range(8):
        pose = vm.look_along_x((0.05 * k, -0.6 + 0.17 * k, 0.02 * k))
        frames.append((scenes.render(cam, pose, boxes), pose))
    _run_pair(cfg, frames)


@pytest.mark.parametrize("vox_inf,depth_m", [(0, 6.5), (2, 5.0)])
def test_pipeline_cfg1_cfg2_640x480(gpu_lib, vox_inf, depth_m):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, depth_m)
    grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=depth_m)
    frames = []
    for k in range(3):
        pose = vm.look_along_x((0.0, 0.11 * k, 0.0))
        frames.append((scenes.render(cam, pose, scenes.box_field_boxes(1 + k)), pose))
    frames.append((scenes.stress_depth(cam, seed=1), vm.look_along_x((0.0, 0.35, 0.0))))
    _run_pair(cfg, frames)


@pytest.mark.parametrize("vox_inf,depth_m", [(0, 6.5), (2, 6.5), (1, 2.2)])
def test_k1_points_on_voxel_faces(gpu_lib, vox_inf, depth_m):
    """Frames of walls at depths that are whole multiples of the voxel size,
    so one coordinate of each of their points lies (within rounding) on a
    voxel face: the fast floor declines there and the near-integer floor or
    the division decides, in the batched K1 (deferred pass), the warps that
    switch to one pixel at a time, and (depth 2.2 m: most walls beyond it) the
    compacting K1."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, depth_m)
    grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=depth_m)
    rng = np.random.default_rng(7 + vox_inf)
    frames = []
    for k, walls in enumerate(((2.0,), (1.5, 3.0), (0.5, 2.5, 4.0, 6.0), (2.0, 4.0, 6.0), (1.0, 2.1, 3.0))):
        d = np.empty((480, 640), np.float32)
        for rows, w in zip(np.array_split(np.arange(480), len(walls)), walls):
            d[rows] = w
        idx = rng.choice(d.size, 2000, replace=False)
        d.flat[idx] = rng.uniform(0.3, 6.0, idx.size).astype(np.float32)
        frames.append((d, vm.look_along_x((0.0, 0.1 * k, 0.0))))
    _run_pair(cfg, frames)


def test_pipeline_cloud_entry_point(gpu_lib):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=4.0)
    gpu = vm.MappingPipeline(cfg)
    orc = oracle_pipeline(cfg)
    rng = np.random.default_rng(5)
    for k in range(4):
        n = int(rng.integers(0, 3000))
        xs, ys, zs = rng.uniform(-3, 3, n), rng.uniform(-2, 2, n), rng.uniform(0.1, 6, n)
        pose = (random_rotation(rng), rng.uniform(-0.3, 0.3, 3))
        sg = gpu.integrate(xs, ys, zs, pose)
        sr = orc.integrate(xs, ys, zs, pose)
        for key in ("points_total", "points_outside", "rays_traced", "voxels_freed",
                    "voxels_marked_unknown_traced", "occupied_count", "freed_count", "shifted"):
            assert sg[key] == sr[key], (k, key)
        assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0])


def test_pipeline_rejects_invalid_transform(gpu_lib):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 64, 48, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    gpu = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=0, depth=4.0))
    with pytest.raises(ValueError, match="invalid transform"):
        gpu.integrate_depth(np.ones((48, 64), np.float32), (2.0 * np.eye(3), np.zeros(3)))


def test_batched_streams_equal_independent_pipelines(gpu_lib):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=6.5)
    S = 5
    batch = vm.MappingPipeline(cfg, n_streams=S)
    singles = [oracle_pipeline(cfg) for _ in range(S)]
    for k in range(4):
        poses = [vm.look_along_x((0.02 * s, 0.09 * k * (s + 1) - 0.2, 0.0)) for s in range(S)]
        depth = np.stack([scenes.render(cam, poses[s], scenes.box_field_boxes(1 + s)) for s in range(S)])
        stats = batch.integrate_depth(depth, poses)
        for s in range(S):
            sr = singles[s].integrate_depth(depth[s], poses[s])
            assert stats[s]["occupied_count"] == sr["occupied_count"]
            assert stats[s]["voxels_freed"] == sr["voxels_freed"]
            assert np.array_equal(batch.local_grid(s)[0], singles[s].local_grid()[0]), (k, s)


@pytest.mark.parametrize("vox_inf,extent", [(1, (6.0, 6.0, 3.0)), (3, (6.4, 5.0, 2.8)), (6, (9.6, 4.5, 3.0)),
                                             (2, (6.2, 5.0, 2.0))])
def test_batched_dilation_radii(gpu_lib, vox_inf, extent):
    """The batch dilation (8x8 tiles; one warp per tile row walking its z
    column when rows fit a warp) for compiled radii 1-4, the run-time radius
    path (6) and a row length that is not a multiple of 4 (62 cells)."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 96, 72, 5.0)
    grid = vm.GridSpec.create_centered(*extent, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=5.0)
    S = 4
    batch = vm.MappingPipeline(cfg, n_streams=S)
    singles = [oracle_pipeline(cfg) for _ in range(S)]
    for k in range(3):
        poses = [vm.look_along_x((0.07 * k * s, 0.1 * k - 0.1 * s, 0.03 * s)) for s in range(S)]
        depth = np.stack([scenes.render(cam, poses[s], scenes.box_field_boxes(1 + s)) for s in range(S)])
        stats = batch.integrate_depth(depth, poses)
        for s in range(S):
            sr = singles[s].integrate_depth(depth[s], poses[s])
            assert stats[s]["occupied_count"] == sr["occupied_count"], (k, s)
            assert np.array_equal(batch.local_grid(s)[0], singles[s].local_grid()[0]), (k, s)


@pytest.mark.parametrize("clear", [False, True], ids=["epoch_keys", "clear_keys"])
def test_long_rows_direct_merge_x_shifts(gpu_lib, clear):
    """Rows longer than 128 cells (200, 204) through the direct-load K4: flat
    chunks for frames that shift only along y, the per-row loop for frames
    that shift along x; both key formats."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 96, 72, 6.0)
    for extent in ((20.0, 4.0, 2.0), (20.4, 3.0, 1.6)):
        grid = vm.GridSpec.create_centered(*extent, 0.1, (0.0, 0.0, 0.0))
        cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.0)
        S = 3
        batch = vm.MappingPipeline(cfg, n_streams=S, flags=N.FLAG_CLEAR_KEYS if clear else 0)
        singles = [oracle_pipeline(cfg) for _ in range(S)]
        for k in range(4):
            poses = [vm.look_along_x((0.23 * k * (s - 1), 0.12 * k, 0.0)) for s in range(S)]
            depth = np.stack([scenes.render(cam, poses[s], scenes.box_field_boxes(1 + s)) for s in range(S)])
            stats = batch.integrate_depth(depth, poses)
            for s in range(S):
                sr = singles[s].integrate_depth(depth[s], poses[s])
                for key in ("occupied_count", "freed_count", "shift_offset"):
                    assert stats[s][key] == sr[key], (extent, k, s, key)
                assert np.array_equal(batch.local_grid(s)[0], singles[s].local_grid()[0]), (extent, k, s)
        batch.close()


def test_large_batch_x_shifts(gpu_lib):
    """A batch large enough for the merge grid's 16 rows per warp (32
    streams of a 100x100x50 grid: four 4-row groups per warp in the row-path
    K4, several 16-cell chunks per thread in the flat K4) with diagonal
    motion, so frames shift along x (row path) and along y only (flat)."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 5.0)
    grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0)
    S = 32
    batch = vm.MappingPipeline(cfg, n_streams=S)
    singles = [oracle_pipeline(cfg) for _ in range(S)]
    for k in range(4):
        poses = [vm.look_along_x((0.13 * k * (s % 3), 0.11 * k * (s % 4) - 0.2, 0.0)) for s in range(S)]
        depth = np.stack([scenes.render(cam, poses[s], scenes.box_field_boxes(1 + s % 3)) for s in range(S)])
        stats = batch.integrate_depth(depth, poses)
        for s in range(S):
            sr = singles[s].integrate_depth(depth[s], poses[s])
            for key in ("occupied_count", "freed_count", "voxels_freed", "shift_offset", "origin"):
                assert stats[s][key] == sr[key], (k, s, key)
            assert np.array_equal(batch.local_grid(s)[0], singles[s].local_grid()[0]), (k, s)


def test_pipeline_long_trajectory_wraps_epochs(gpu_lib):
    """cfg4-style moving robot over more frames than the 8-bit epoch holds
    (255), shifting by about one voxel per frame."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 64, 48, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, -8.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    boxes = scenes.corridor_boxes(-12.0, 25.0)
    gpu = vm.MappingPipeline(cfg)
    orc = oracle_pipeline(cfg)
    shifts = 0
    for k in range(300):
        pose = vm.look_along_x((0.0, -8.0 + 0.1001 * k, 0.0))
        depth = scenes.render(cam, pose, boxes)
        sg = gpu.integrate_depth(depth, pose)
        sr = orc.integrate_depth(depth, pose)
        shifts += sr["shifted"]
        for key in ("occupied_count", "freed_count", "voxels_freed", "voxels_marked_unknown_traced",
                    "shifted", "shift_offset", "origin", "points_outside"):
            assert sg[key] == sr[key], (k, key, sg[key], sr[key])
        if k % 50 == 49 or k == 299:
            assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0]), k
    assert shifts > 250


@pytest.mark.parametrize("flags", [0, 8], ids=["default", "no_tma_merge"])
@pytest.mark.parametrize("extent,vox,motion", [((5.0, 3.0, 2.0), 0.1, (1.0, 0.6, -0.4)),
                                               ((10.0, 3.0, 2.0), 0.05, (1.0, 0.6, -0.4)),
                                               ((3.3, 2.0, 1.5), 0.1, (1.0, 0.6, -0.4)),
                                               ((6.4, 3.2, 1.6), 0.1, (1.0, 0.6, -0.4)),
                                               ((6.4, 3.2, 1.6), 0.1, (0.0, 1.0, -0.7)),
                                               ((6.4, 3.2, 1.6), 0.1, (0.0, -0.3, 1.0)),
                                               ((10.0, 3.0, 2.0), 0.05, (0.0, 1.0, 0.5))],
                         ids=["dx50", "dx200", "dx33", "dx64", "dx64-yz", "dx64-zy", "dx200-yz"])
def test_k4_variants_diagonal_motion(gpu_lib, flags, extent, vox, motion):
    """The K4 variants (TMA-staged rows for long / odd rows; direct loads for
    short word-aligned rows, with 16-cell flat chunks when the frame has no x
    shift; flag 8 forces the direct kernel) against the reference while the
    robot drifts, so the grid shifts by one or two voxels per frame, in x by
    amounts that are not multiples of 4, or only in y and z."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 64, 48, 6.5)
    grid = vm.GridSpec.create_centered(*extent, vox, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    boxes = scenes.box_field_boxes(3)
    gpu = vm.MappingPipeline(cfg, flags=flags)
    orc = oracle_pipeline(cfg)
    for k in range(24):
        step = 1.37 * vox * k
        pose = vm.look_along_x(tuple(m * step for m in motion))
        depth = scenes.render(cam, pose, boxes)
        sg = gpu.integrate_depth(depth, pose)
        sr = orc.integrate_depth(depth, pose)
        for key in ("occupied_count", "freed_count", "shifted", "shift_offset", "origin"):
            assert sg[key] == sr[key], (k, key, sg[key], sr[key])
        assert np.array_equal(gpu.local_grid()[0], orc.local_grid()[0]), k


def test_async_double_buffered_host_path(gpu_lib):
    """vxm_integrate_depth_async: queued host frames (pinned) give the same
    grids as the synchronous path and the reference."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=6.5)
    S, F = 3, 6
    poses = [[vm.look_along_x((0.01 * s, 0.08 * k - 0.2, 0.0)) for s in range(S)] for k in range(F)]
    frames = [np.stack([scenes.render(cam, poses[k][s], scenes.box_field_boxes(1 + s)) for s in range(S)])
              for k in range(F)]
    pinned = [torch.from_numpy(f).pin_memory() for f in frames]
    pipe = vm.MappingPipeline(cfg, n_streams=S)
    for k in range(F):
        pipe.integrate_depth_async(pinned[k].data_ptr(), poses[k])
    last = pipe.wait_stats()
    refs = [oracle_pipeline(cfg) for _ in range(S)]
    for s in range(S):
        for k in range(F):
            sr = refs[s].integrate_depth(frames[k][s], poses[k][s])
        assert last[s]["freed_count"] == sr["freed_count"]
        assert np.array_equal(pipe.local_grid(s)[0], refs[s].local_grid()[0]), s


def test_snapshot_save_resume_matches_uninterrupted(gpu_lib, tmp_path):
    """Checkpoint/resume through VOXGRID1 files: a pipeline
    resumed from a snapshot continues exactly like the uninterrupted one, and
    the snapshot file equals the reference's write_grid of the same grid."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 96, 72, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5)
    boxes = scenes.box_field_boxes(2)
    poses = [vm.look_along_x((0.05 * k, 0.12 * k - 0.4, 0.0)) for k in range(10)]
    frames = [scenes.render(cam, p, boxes) for p in poses]
    full = vm.MappingPipeline(cfg, n_streams=2)
    for k in range(5):
        full.integrate_depth(np.stack([frames[k]] * 2), [poses[k]] * 2)
    snap = tmp_path / "s1.vox"
    full.save_snapshot(snap, s=1)
    cells, origin = full.local_grid(1)
    g = vm.GridSpec.create(6.0, 6.0, 3.0, 0.1, origin)
    ref.write_grid(g.c, cells, tmp_path / "ref.vox")
    assert snap.read_bytes() == (tmp_path / "ref.vox").read_bytes()
    resumed = vm.MappingPipeline(cfg)
    resumed.load_snapshot(snap)
    for k in range(5, 10):
        sf = full.integrate_depth(np.stack([frames[k]] * 2), [poses[k]] * 2)[1]
        sr = resumed.integrate_depth(frames[k], poses[k])
        assert sf["freed_count"] == sr["freed_count"] and sf["origin"] == sr["origin"], k
    assert np.array_equal(full.local_grid(1)[0], resumed.local_grid()[0])
    bad = vm.MappingPipeline(vm.PipelineConfig(vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0, 0, 0)),
                                               cam, vox_inf=1, depth=6.5))
    with pytest.raises(ValueError, match="does not match"):
        bad.load_snapshot(snap)


def test_branched_batch_equals_single_streams(gpu_lib):
    """Batches of >= 12 streams run as graph branches over stream shares
    (13 streams: shares 4/4/5); every stream must equal its own single-stream
    pipeline, and one of them the reference."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 96, 72, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=6.0)
    S = 13
    batch = vm.MappingPipeline(cfg, n_streams=S)
    assert batch.graph_branches == 3
    single = vm.MappingPipeline(cfg, n_streams=S, flags=4)  # VXM_FLAG_SINGLE_BRANCH
    assert single.graph_branches == 1
    ones = [vm.MappingPipeline(cfg) for _ in range(S)]
    orc = oracle_pipeline(cfg)
    for k in range(4):
        poses = [vm.look_along_x((0.03 * s, 0.11 * k - 0.2, 0.01 * s)) for s in range(S)]
        depth = np.stack([scenes.render(cam, poses[s], scenes.box_field_boxes(1 + s % 4)) for s in range(S)])
        sb = batch.integrate_depth(depth, poses)
        ss = single.integrate_depth(depth, poses)
        so = orc.integrate_depth(depth[7], poses[7])
        for s in range(S):
            s1 = ones[s].integrate_depth(depth[s], poses[s])
            for key in ("occupied_count", "freed_count", "voxels_freed", "voxels_marked_unknown_traced",
                        "points_total", "origin"):
                assert sb[s][key] == s1[key] == ss[s][key], (k, s, key)
        assert sb[7]["freed_count"] == so["freed_count"]
    for s in range(S):
        assert np.array_equal(batch.local_grid(s)[0], ones[s].local_grid()[0]), s
    assert np.array_equal(batch.local_grid(7)[0], orc.local_grid()[0])


@pytest.mark.parametrize("shape", [(63, 47), (61, 40), (66, 49)])
def test_pipeline_odd_frame_shapes_and_special_depths(gpu_lib, shape):
    """W*H not a multiple of 4 (K1 without the TMA staging), rows that end
    inside a 4-pixel quad, and depth values the validity test must reject:
    NaN, +-inf, negative, -0, subnormal, exactly max_depth and just above."""
    W, H = shape
    cam = vm.CameraModel(85 * DEG, 101 * DEG, W, H, 5.0)
    grid = vm.GridSpec.create_centered(6.0, 5.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=5.0)
    rng = np.random.default_rng(W * H)
    frames = []
    for k in range(3):
        pose = vm.look_along_x((0.0, 0.13 * k, 0.02 * k))
        d = scenes.render(cam, pose, scenes.box_field_boxes(2 + k)).copy()
        special = np.array([np.nan, np.inf, -np.inf, -1.0, -0.0, 1e-40, 5.0, np.nextafter(np.float32(5.0), 10),
                            0.0, 4.9999995], dtype=np.float32)
        idx = rng.choice(d.size, 200, replace=False)
        d.flat[idx] = special[rng.integers(0, special.size, idx.size)]
        frames.append((d, pose))
    frames.append((scenes.stress_depth(cam, seed=3, invalid=0.3), vm.look_along_x((0.0, 0.4, 0.0))))
    _run_pair(cfg, frames)


@pytest.mark.parametrize("max_depth", [5.0, 4.7, 6.3])
def test_pipeline_compacting_k1_special_depths(gpu_lib, max_depth):
    """The compacting, TMA-staged K1 (W*H % 4 == 0, sparse frames): its depth
    test compares floats against the largest float <= max_depth, which must
    equal the reference's double comparison (geometry.cpp:53-54) also when
    max_depth is not a float; NaN, +-inf, zero, negative, subnormal depths and
    the floats either side of max_depth."""
    W, H = 96, 64
    cam = vm.CameraModel(85 * DEG, 101 * DEG, W, H, max_depth)
    grid = vm.GridSpec.create_centered(8.0, 8.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=min(max_depth, 4.5))
    rng = np.random.default_rng(int(max_depth * 10))
    m32 = np.float32(max_depth)
    near = [np.nextafter(m32, np.float32(0)), m32, np.nextafter(m32, np.float32(100)),
            np.nextafter(np.nextafter(m32, np.float32(100)), np.float32(100))]
    special = np.array([np.nan, np.inf, -np.inf, -1.0, -0.0, 0.0, 1e-40] + near, dtype=np.float32)
    frames = []
    for k in range(6):
        pose = vm.look_along_x((0.0, 0.11 * k, 0.0))
        d = scenes.render(cam, pose, scenes.box_field_boxes(1)).copy()
        d[rng.random(d.shape) < 0.6] = 0.0  # sparse: the host switches to the compacting K1
        idx = rng.choice(d.size, 600, replace=False)
        d.flat[idx] = special[rng.integers(0, special.size, idx.size)]
        frames.append((d, pose))
    _run_pair(cfg, frames)


def test_per_pixel_tracer_branched_batch(gpu_lib):
    """TracerMode::PerPixelBaseline in a batch big enough for graph branches."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 80, 60, 6.5)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.5, tracer_mode=1)
    S = 12
    batch = vm.MappingPipeline(cfg, n_streams=S)
    assert batch.graph_branches == 3
    orc = [oracle_pipeline(cfg) for _ in (0, 11)]
    for k in range(3):
        poses = [vm.look_along_x((0.02 * s, 0.1 * k, 0.0)) for s in range(S)]
        depth = np.stack([scenes.render(cam, poses[s], scenes.box_field_boxes(1 + s % 3)) for s in range(S)])
        st = batch.integrate_depth(depth, poses)
        for o, s in zip(orc, (0, 11)):
            sr = o.integrate_depth(depth[s], poses[s])
            assert st[s]["voxels_freed"] == sr["voxels_freed"] and st[s]["freed_count"] == sr["freed_count"]
    for o, s in zip(orc, (0, 11)):
        assert np.array_equal(batch.local_grid(s)[0], o.local_grid()[0])


def test_stage_times_from_kernel_stamps(gpu_lib):
    """vxm_stats::*_us come from the kernels' %globaltimer stamps (no event
    nodes in the frame graph): positive for every stage, shift_us 0, and the
    graph-timed frame brackets their sum."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 5.0)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    pipe = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0))
    pose = vm.look_along_x((0.0, 0.0, 0.0))
    depth = scenes.render(cam, pose, scenes.box_field_boxes(1))
    for _ in range(3):
        st = pipe.integrate_depth(depth, pose)
    assert st["populate_us"] > 0.0 and st["trace_us"] > 0.0 and st["merge_us"] > 0.0
    assert st["shift_us"] == 0.0
    assert st["populate_us"] + st["trace_us"] + st["merge_us"] <= pipe.last_frame_ms() * 1000.0 + 1.0


def test_stage_events_attached_to_graph(gpu_lib):
    """Caller events recorded at the stage boundaries inside the frame graph
    (VXM_FLAG_STAGE_EVENTS; the bench's kernel-timing pass) time the stages
    in order, and the results equal a pipeline without them."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 5.0)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0)
    S = 12
    poses = [vm.look_along_x((0.0, 0.05 * s, 0.0)) for s in range(S)]
    depth = vm.render_depth(cam, poses, scenes.box_field_boxes(2))
    dev = torch.from_numpy(depth).cuda()
    timed = vm.MappingPipeline(cfg, n_streams=S, flags=vm.N.FLAG_STAGE_EVENTS | vm.N.FLAG_SINGLE_BRANCH)
    plain = vm.MappingPipeline(cfg, n_streams=S)
    stream = torch.cuda.ExternalStream(timed.cuda_stream)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in evs:
        e.record(stream)
    timed.set_stage_events([e.cuda_event for e in evs])
    pa = vm.pose_array(poses)
    for _ in range(2):
        timed.integrate_depth_device(dev.data_ptr(), pa)
        st_t = timed.wait_stats()
        plain.integrate_depth_device(dev.data_ptr(), pa)
        st_p = plain.wait_stats()
    torch.cuda.synchronize()
    spans = [evs[i].elapsed_time(evs[i + 1]) for i in range(3)]
    assert all(t > 0.0 for t in spans), spans
    timed.set_stage_events(None)
    for s in range(S):
        for key in ("occupied_count", "freed_count", "voxels_freed", "rays_traced"):
            assert st_t[s][key] == st_p[s][key]
        assert np.array_equal(timed.local_grid(s)[0], plain.local_grid(s)[0])


@pytest.mark.parametrize("path,S", [("device", 12), ("async", 12), ("host", 12), ("device", 13)])
def test_desynchronised_batch_across_epoch_wrap(gpu_lib, path, S):
    """A batch of 12 streams runs as three per-branch graphs on their own
    streams (each waiting only for its call's inputs); 300 back-to-back calls
    cross the 8-bit epoch wrap, whose array clears go on the owning branch's
    stream. Every stream ends equal to an independent single-stream pipeline
    (and to the per-call joined-branch form, VXM_FLAG_NO_DESYNC)."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 48, 36, 6.5)
    grid = vm.GridSpec.create_centered(4.0, 4.0, 2.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=1, depth=6.0)
    calls = 300
    boxes = scenes.box_field_boxes(4)
    poses = [[vm.look_along_x((0.03 * (k % 40), 0.02 * s + 0.01 * (k % 17), 0.0)) for s in range(S)]
             for k in range(12)]
    frames = [vm.render_depth(cam, poses[k], boxes) for k in range(12)]
    pa = [vm.pose_array(poses[k]) for k in range(12)]
    batch = vm.MappingPipeline(cfg, n_streams=S)
    joined = vm.MappingPipeline(cfg, n_streams=S, flags=vm.N.FLAG_NO_DESYNC)
    singles = [vm.MappingPipeline(cfg) for _ in (0, S - 1)]
    dev = [torch.from_numpy(f).cuda() for f in frames]
    pinned = [torch.from_numpy(f).pin_memory() for f in frames]
    for k in range(calls):
        q = k % 12
        if path == "device":
            batch.integrate_depth_device(dev[q].data_ptr(), pa[q])
        elif path == "async":
            batch.integrate_depth_async(pinned[q].data_ptr(), pa[q])
        else:
            batch.integrate_depth_ptr(pinned[q].data_ptr(), pa[q])
        joined.integrate_depth_device(dev[q].data_ptr(), pa[q])
        for i, s in enumerate((0, S - 1)):
            singles[i].integrate_depth(frames[q][s], poses[q][s])
    st = batch.wait_stats()
    sj = joined.wait_stats()
    for s in range(S):
        assert st[s]["freed_count"] == sj[s]["freed_count"]
        assert np.array_equal(batch.local_grid(s)[0], joined.local_grid(s)[0]), s
    for i, s in enumerate((0, S - 1)):
        assert np.array_equal(batch.local_grid(s)[0], singles[i].local_grid()[0]), s


def test_device_frames_produced_on_another_stream(gpu_lib):
    """Frames written by the caller on its own stream right before the call:
    vxm_set_input_event makes the (desynchronised) batch wait for them."""
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 5.0)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0)
    S = 12
    poses = [vm.look_along_x((0.0, 0.05 * s, 0.0)) for s in range(S)]
    frames = vm.render_depth(cam, poses, scenes.box_field_boxes(3))
    host = torch.from_numpy(frames).pin_memory()
    dev = torch.empty_like(host, device="cuda")
    producer = torch.cuda.Stream()
    pipe = vm.MappingPipeline(cfg, n_streams=S)
    ref = vm.MappingPipeline(cfg, n_streams=S)
    pa = vm.pose_array(poses)
    for k in range(3):
        with torch.cuda.stream(producer):
            dev.zero_()
            torch.cuda._sleep(2_000_000)  # a slow producer
            dev.copy_(host, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(producer)
        pipe.set_input_event(ready.cuda_event)
        pipe.integrate_depth_device(dev.data_ptr(), pa)
        st = pipe.wait_stats()
        sr = ref.integrate_depth(frames, poses)
        for s in range(S):
            assert st[s]["points_total"] == sr[s]["points_total"]
            assert st[s]["freed_count"] == sr[s]["freed_count"]
    for s in range(S):
        assert np.array_equal(pipe.local_grid(s)[0], ref.local_grid(s)[0])


@pytest.mark.parametrize("dims_cells", [(159, 21, 9), (133, 17, 7), (201, 13, 5)])
def test_tma_merge_odd_rows_two_stages(gpu_lib, dims_cells):
    """TMA-staged K4 with row groups whose stage size is not a multiple of
    16 bytes (found by tools/fuzz_parity.py: 159-cell rows): the second stage
    buffer stays 16-byte aligned. A moving robot, batch of 13 streams."""
    vox = 0.1
    grid = vm.GridSpec.create_centered(*(d * vox for d in dims_cells), vox, (0.0, 0.0, 0.0))
    assert tuple(grid.dims) == dims_cells
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 40, 32, 6.0)
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=6.0)
    S = 13
    gpu = vm.MappingPipeline(cfg, n_streams=S)
    refs = [oracle_pipeline(cfg) for _ in (0, S - 1)]
    boxes = scenes.box_field_boxes(6)
    for k in range(6):
        poses = [vm.look_along_x((0.13 * k + 0.02 * s, -0.07 * k, 0.05 * k)) for s in range(S)]
        depth = vm.render_depth(cam, poses, boxes)
        st = gpu.integrate_depth(depth, poses)
        for i, s in enumerate((0, S - 1)):
            sr = refs[i].integrate_depth(depth[s], poses[s])
            assert st[s]["freed_count"] == sr["freed_count"] and st[s]["occupied_count"] == sr["occupied_count"]
    for i, s in enumerate((0, S - 1)):
        assert np.array_equal(gpu.local_grid(s)[0], refs[i].local_grid()[0])
