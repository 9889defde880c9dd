"""The reference's own pipeline test cases and acceptance criteria
(proj/tests/test_pipeline.cpp, proj/tests/acceptance.cpp), run against two
backends: the plain-C oracle (CPU) and the sm_100a path through the C-ABI
(GPU). Known answers are the reference's; the criterion-9 Free counts are the
numbers its recorded run printed (proj/test_output.txt:29)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import c_oracle as co
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes

DEG = math.pi / 180.0
BACKENDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


def make(backend, cfg):
    if backend == "oracle":
        return co.Pipeline(cfg.to_c())
    return vm.MappingPipeline(cfg)


def small_config(tracer=vm.N.TRACER_BUNDLED):
    # test_pipeline.cpp:15-24
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0.0, 0.0, 0.0))
    return vm.PipelineConfig(grid, vm.CameraModel(85 * DEG, 101 * DEG, 320, 240, 6.5), vox_inf=0, depth=4.0,
                             tracer_mode=tracer)


def wall_cloud(depth):
    # test_pipeline.cpp:28-36: 57x57 points, 5 cm apart
    i = np.arange(-28, 29) * 0.05
    xs, ys = np.meshgrid(i, i)  # j outer, i inner
    return xs.ravel().copy(), ys.ravel().copy(), np.full(xs.size, depth)


def cell(cells, x, y, z, dims=(40, 40, 20)):
    return int(cells[x + y * dims[0] + z * dims[0] * dims[1]])


@pytest.fixture(params=BACKENDS)
def backend(request):
    if request.param == "gpu":
        from paper_2112_13169_b200 import _native
        if _native.load().vxm_device_count() == 0:
            pytest.fail("no sm_100 device for a gpu test")
    return request.param


def test_empty_frame_carves_free_space(backend):
    cfg = small_config()
    p = make(backend, cfg)
    st = p.integrate(np.zeros(0), np.zeros(0), np.zeros(0), vm.look_along_x((0, 0, 0)))
    vd, vw, vh = vm.bundle_dimensions(cfg.camera, cfg.depth, 0.15)
    assert st["points_total"] == 0
    assert st["rays_traced"] == vw * vh
    assert st["voxels_marked_unknown_traced"] == 0
    assert st["occupied_count"] == 0 and st["freed_count"] > 0 and not st["shifted"]
    cells, _ = p.local_grid()
    assert int((cells == 3).sum()) == 0
    assert int((cells == 1).sum()) == st["freed_count"]


def test_wall_frame_free_occupied_unknown_in_depth_order(backend):
    p = make(backend, small_config())
    st = p.integrate(*wall_cloud(2.0), vm.look_along_x((0, 0, 0)))
    cells, _ = p.local_grid()
    assert st["occupied_count"] > 0 and st["voxels_marked_unknown_traced"] > 0
    assert int((cells == 3).sum()) == 0
    assert all(cell(cells, x, 20, 10) == 1 for x in range(21, 33))
    assert cell(cells, 33, 20, 10) == 2
    assert all(cell(cells, x, 20, 10) == 0 for x in range(34, 40))
    # outside the frustum nothing is touched (camera at x = 20 looking +x)
    g = cells.reshape(20, 40, 40)
    assert int(g[:, :, :20].max()) == 0
    assert st["occupied_count"] == int((cells == 2).sum())
    assert st["freed_count"] == int((cells == 1).sum())
    assert st["points_total"] == 57 * 57


def test_receding_wall_clears_old_footprint(backend):
    p = make(backend, small_config())
    p.integrate(*wall_cloud(2.0), vm.look_along_x((0, 0, 0)))
    assert cell(p.local_grid()[0], 33, 20, 10) == 2
    p.integrate(*wall_cloud(2.75), vm.look_along_x((0, 0, 0)))
    cells, _ = p.local_grid()
    assert cell(cells, 33, 20, 10) == 1
    assert cell(cells, 38, 20, 10) == 2


def test_recenters_once_the_camera_drifts_a_voxel(backend):
    cfg = small_config()
    p = make(backend, cfg)
    st = p.integrate(np.zeros(0), np.zeros(0), np.zeros(0), vm.look_along_x((0.05, 0, 0)))
    assert not st["shifted"]
    assert np.allclose(p.local_grid()[1], cfg.grid.origin)
    st = p.integrate(np.zeros(0), np.zeros(0), np.zeros(0), vm.look_along_x((0.4, 0, 0)))
    assert st["shifted"] and tuple(st["shift_offset"]) == (3, 0, 0)
    assert np.allclose(p.local_grid()[1], cfg.grid.origin + np.array([3 * 0.15, 0, 0]))


def test_invalid_pose_is_rejected(backend):
    p = make(backend, small_config())
    with pytest.raises(ValueError):
        p.integrate(np.zeros(0), np.zeros(0), np.zeros(0), (2.0 * np.eye(3), np.zeros(3)))


def test_dynamic_obstacle_criterion_12(backend):
    # acceptance.cpp:430-486: occluded cells Unknown, then Free once vacated
    p = make(backend, small_config())
    p.integrate(*wall_cloud(2.0), vm.look_along_x((0, 0, 0)))
    first, _ = p.local_grid()
    assert cell(first, 33, 20, 10) == 2
    assert all(cell(first, x, 20, 10) == 0 for x in range(34, 39))
    p.integrate(*wall_cloud(2.75), vm.look_along_x((0, 0, 0)))
    second, _ = p.local_grid()
    assert cell(second, 33, 20, 10) == 1
    assert all(cell(second, x, 20, 10) == 1 for x in range(34, 38))
    assert cell(second, 38, 20, 10) == 2


@pytest.mark.parametrize("scene,tracer,expect", [
    ("wall", vm.N.TRACER_BUNDLED, 29712), ("wall", vm.N.TRACER_PER_PIXEL, 28900),
    ("boxes", vm.N.TRACER_BUNDLED, 32613), ("boxes", vm.N.TRACER_PER_PIXEL, 39082)])
def test_criterion_9_recorded_free_counts(backend, scene, tracer, expect):
    """compare_methods (proj/src/sim/bench.cpp:225-290) as acceptance
    criterion 9 runs it (acceptance.cpp:340-371): default AppConfig,
    Sequential, vox_inf 0, 5-frame strafe (0,-0.6,0) -> (0,0.6,0); the final
    Free counts are the reference's recorded ones (proj/test_output.txt:29)."""
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 320, 240, 6.5)
    grid = vm.GridSpec.create_centered(15.0, 15.0, 3.0, 0.15, (0.0, -0.6, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=0, depth=6.5, tracer_mode=tracer)
    p = make(backend, cfg)
    boxes = scenes.wall_boxes(5.5) if scene == "wall" else scenes.box_field_boxes(109)
    for f in range(5):
        pose = vm.look_along_x((0.0, -0.6 + (f / 4) * 1.2, 0.0))
        p.integrate_depth(scenes.render(cam, pose, boxes), pose)
    cells, _ = p.local_grid()
    assert int((cells == 1).sum()) == expect
