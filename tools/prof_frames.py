"""A few frames of cfg1/cfg2 (S=1 and S=64) for ncu launch lists."""
import math, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
which = sys.argv[1] if len(sys.argv) > 1 else "all"
for name, vox_inf, dm, S in (("cfg1", 0, 6.5, 1), ("cfg2", 2, 5.0, 1), ("cfg2x64", 2, 5.0, 64)):
    if which != "all" and which != name:
        continue
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, dm)
    grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0, 0, 0))
    p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=dm), n_streams=S, flags=2)
    pose = vm.look_along_x((0, 0, 0))
    d = scenes.render(cam, pose, scenes.box_field_boxes(1))
    dev = torch.from_numpy(np.stack([d] * S)).cuda()
    for _ in range(6):
        p.integrate_depth_device(dev.data_ptr(), [pose] * S); p.wait_stats()
