"""cfg4 at full size (BASELINE.json configs[3]): the 1000-frame
sweep_trajectory((0,-50,0),(0,50,0),1000) (proj/src/sim/trajectory.cpp:15-25)
on cfg1 frames (640x480, 0.1 m voxels, 100x100x50 grid, 6.5 m) through the
corridor scene, about one local-grid shift per frame. Every frame's stats and
every 50th grid against the reference's Sequential pipeline, through the
single-frame path and the multi-frame path (64 frames per call, chain-folded
merge). Frames come from the GPU renderer (bit-identical to the reference's
render_depth, tests/test_gpu_render.py) and are fed to both sides."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests import workload as W
from tests.oracle_api import have_ref, oracle_pipeline

pytestmark = pytest.mark.gpu

if not have_ref():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

KEYS = ("points_total", "points_outside", "rays_traced", "voxels_freed", "voxels_marked_unknown_traced",
        "voxels_skipped_out_of_bounds", "occupied_count", "freed_count", "shifted", "shift_offset", "origin")


def test_cfg4_full_size_1000_frame_sweep(gpu_lib):
    import torch

    c = W.CONFIGS["cfg1"]
    cam = W.camera(vm, c)
    positions = W.sweep_positions(1000)
    poses = [vm.look_along_x(p) for p in positions]
    cfg = vm.PipelineConfig(W.grid_for(vm, c, positions[0]), cam, vox_inf=0, depth=c["depth"])
    assert cfg.grid.dims == (100, 100, 50)
    boxes = scenes.corridor_boxes(-60.0, 60.0)
    one = vm.MappingPipeline(cfg)
    F = 64
    seq = vm.MappingPipeline(cfg, frames_per_call=F)
    orc = oracle_pipeline(cfg)
    shifts = 0
    for i0 in range(0, 1000, F):
        n = min(F, 1000 - i0)
        chunk = poses[i0:i0 + n]
        depth = vm.render_depth(cam, chunk, boxes)
        if n == F:
            dev = torch.from_numpy(depth).cuda()
            seq.integrate_depth_device(dev.data_ptr(), vm.pose_array(chunk))
            sq = seq.wait_stats()
        else:
            sq = seq.integrate_depth_frames(depth, chunk)
        for j in range(n):
            i = i0 + j
            sr = orc.integrate_depth(depth[j], chunk[j])
            sg = one.integrate_depth(depth[j], chunk[j])
            shifts += sr["shifted"]
            for key in KEYS:
                assert sg[key] == sr[key], (i, key, sg[key], sr[key])
                assert sq[j][key] == sr[key], ("seq", i, key, sq[j][key], sr[key])
            if i % 50 == 49 or i == 999:
                rc = orc.local_grid()[0]
                assert np.array_equal(one.local_grid()[0], rc), i
        assert np.array_equal(seq.local_grid()[0], orc.local_grid()[0]), i0
    assert shifts > 700  # the reference recentres on 749 of the 1000 frames
