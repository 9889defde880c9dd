"""Scratch timing of the per-frame graph (device-resident depth), cfg1/cfg2."""
import math, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
for name, vox_inf, dm, S in (("cfg1", 0, 6.5, 1), ("cfg2", 2, 5.0, 1), ("cfg2x64", 2, 5.0, 64), ("cfg1x64", 0, 6.5, 64)):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, dm)
    grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0, 0, 0))
    p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=dm), n_streams=S)
    pose = vm.look_along_x((0, 0, 0))
    d = scenes.render(cam, pose, scenes.box_field_boxes(1))
    dev = torch.from_numpy(np.stack([d] * S)).cuda()
    poses = [pose] * S
    for _ in range(5):
        p.integrate_depth_device(dev.data_ptr(), poses); p.wait_stats()
    ts = []
    for k in range(200):
        p.integrate_depth_device(dev.data_ptr(), poses); st = p.wait_stats(); ts.append(p.last_frame_ms())
    ts = np.array(ts)
    print(name, "S", S, "p50 ms %.4f p99 %.4f  frames/s %.0f" % (np.median(ts), np.percentile(ts, 99), S / np.median(ts) * 1e3), st[0]["voxels_freed"], st[0]["occupied_count"], flush=True)
