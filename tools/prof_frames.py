"""A few frames of cfg1/cfg2 (S=1 and S=64), cfg3 (S=8), cfg2 frames on a grid
with 101-cell x-rows (odd8, S=8: the TMA-staged K4) and one 64-frame
moving-robot call (seq64) for ncu launch lists and captures."""
import math, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
which = sys.argv[1] if len(sys.argv) > 1 else "all"
for name, vox_inf, dm, S, F in (("cfg1", 0, 6.5, 1, 1), ("cfg1x64", 0, 6.5, 64, 1), ("cfg2", 2, 5.0, 1, 1), ("cfg2x64", 2, 5.0, 64, 1),
                                ("seq64", 2, 5.0, 1, 64), ("cfg3x8", 0, 6.5, 8, 1), ("odd8", 2, 5.0, 8, 1)):
    if which != "all" and which != name:
        continue
    if name == "cfg3x8":  # 1280x720, 0.05 m voxels, 200x200x100
        cam = vm.CameraModel(85 * DEG, 101 * DEG, 1280, 720, dm)
        grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.05, (0, 0, 0))
    else:
        cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, dm)
        # odd8: 101 x 100 x 50 cells (rows not word-aligned -> TMA-staged K4)
        grid = vm.GridSpec.create_centered(10.1 if name == "odd8" else 10.0, 10.0, 5.0, 0.1, (0, 0, 0))
    p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=dm), n_streams=S, flags=6,
                           frames_per_call=F)
    pose = vm.look_along_x((0, 0, 0))
    d = scenes.render(cam, pose, scenes.box_field_boxes(1))
    dev = torch.from_numpy(np.stack([d] * (S * F))).cuda()
    poses = [pose] * S if F == 1 else [vm.look_along_x((0, 0.1001 * j, 0)) for j in range(F)]
    for _ in range(6):
        p.integrate_depth_device(dev.data_ptr(), poses); p.wait_stats()
