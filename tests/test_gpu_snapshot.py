"""Asynchronous checkpoints (the reference's VOXGRID1
format, proj/src/grid_io.cpp:14-63): vxm_snapshot_save_async returns at once,
integration continues on the GPU while the grid is copied to pinned memory
and a host thread writes the file, and the file is byte-identical to the
reference's write_grid of the reference pipeline's local grid at the point
the snapshot was taken."""
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


@pytest.mark.parametrize("S", [1, 12])
def test_async_snapshot_while_integrating(gpu_lib, tmp_path, S):
    import torch

    from oracle import ref

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 5.0)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.1, (0.0, 0.0, 0.0))
    cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0)
    frames = 12
    poses = [[vm.look_along_x((0.0, 0.1001 * k + 0.03 * s, 0.0)) for s in range(S)] for k in range(frames)]
    depth = [vm.render_depth(cam, poses[k], scenes.box_field_boxes(3)) for k in range(frames)]
    dev = [torch.from_numpy(d).cuda() for d in depth]
    pa = [vm.pose_array(p) for p in poses]
    gpu = vm.MappingPipeline(cfg, n_streams=S)
    s_snap = S - 1
    orc = oracle_pipeline(cfg)
    for k in range(frames):
        gpu.integrate_depth_device(dev[k].data_ptr(), pa[k])  # back to back, no waits
        orc.integrate_depth(depth[k][s_snap], poses[k][s_snap])
        if k in (4, 9):
            path = tmp_path / f"snap{k}.vox"
            gpu.save_snapshot_async(path, s=s_snap)  # the grid after frame k
            cells, origin = orc.local_grid()
            ref.write_grid(vm.GridSpec.create(*grid.c.size, grid.vox_size, tuple(origin)).c, cells,
                           tmp_path / f"ref{k}.vox")
    gpu.snapshot_wait()
    gpu.wait_stats()
    for k in (4, 9):
        assert (tmp_path / f"snap{k}.vox").read_bytes() == (tmp_path / f"ref{k}.vox").read_bytes(), k
    # the run itself was not disturbed
    assert np.array_equal(gpu.local_grid(s_snap)[0], orc.local_grid()[0])
    # a resumed pipeline continues exactly
    resumed = vm.MappingPipeline(cfg)
    resumed.load_snapshot(tmp_path / "snap9.vox")
    assert np.array_equal(resumed.local_grid()[0], vm.read_grid(tmp_path / "snap9.vox")[1])


def test_async_snapshot_reports_write_errors(gpu_lib, tmp_path):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 32, 24, 5.0)
    grid = vm.GridSpec.create_centered(2.0, 2.0, 1.0, 0.1, (0.0, 0.0, 0.0))
    gpu = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=0, depth=5.0))
    gpu.save_snapshot_async(tmp_path / "missing_dir" / "x.vox")
    with pytest.raises(Exception, match="cannot open"):
        gpu.snapshot_wait()
    gpu.snapshot_wait()  # nothing pending any more
