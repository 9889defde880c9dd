"""In-graph stage times of lone frames from the kernels' %globaltimer stamps
(vxm_stats populate_us / trace_us / merge_us), median over 200 frames."""
import math, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
for name, vox_inf, dm, W, H, vs, ext in (("cfg2", 2, 5.0, 640, 480, 0.1, (10, 10, 5)), ("cfg1", 0, 6.5, 640, 480, 0.1, (10, 10, 5)),
                                         ("cfg3", 0, 6.5, 1280, 720, 0.05, (10, 10, 5))):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, W, H, dm)
    grid = vm.GridSpec.create_centered(*ext, vs, (0, 0, 0))
    pose = vm.look_along_x((0, 0, 0))
    d = torch.from_numpy(scenes.render(cam, pose, scenes.box_field_boxes(1))[None]).cuda()
    p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=dm))
    rows = []
    for k in range(220):
        p.integrate_depth_device(d.data_ptr(), [pose])
        st = p.wait_stats()[0]
        if k >= 20:
            rows.append((st["populate_us"], st["trace_us"], st["merge_us"]))
    m = np.median(np.array(rows), axis=0)
    print(f"{name} lone: populate+dilate {m[0]:.1f} us, trace {m[1]:.1f} us, merge {m[2]:.1f} us (in-graph stamps)", flush=True)
    p.close()
