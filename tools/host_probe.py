"""Host-side cost of one batched call (submission only) vs its device time:
is a back-to-back loop of integrate_depth_device host-bound?"""
import math, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, 5.0)
grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0, 0, 0))
p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0), n_streams=S)
pose = vm.look_along_x((0, 0, 0))
d = scenes.render(cam, pose, scenes.box_field_boxes(1))
dev = torch.from_numpy(np.stack([d] * S)).cuda()
pa = vm.pose_array([pose] * S)
for _ in range(10):
    p.integrate_depth_device(dev.data_ptr(), pa)
p.wait_stats()
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(p.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 200
sub = []
e0.record(st)
t0 = time.perf_counter()
for _ in range(n):
    a = time.perf_counter()
    p.integrate_depth_device(dev.data_ptr(), pa)
    sub.append(time.perf_counter() - a)
t1 = time.perf_counter()
e1.record(st)
p.wait_stats()
torch.cuda.synchronize()
print(f"S={S}: host submit per call p50 {np.median(sub)*1e3:.4f} ms max {np.max(sub)*1e3:.3f}; "
      f"loop wall {((t1-t0)/n)*1e3:.4f} ms/call; device {e0.elapsed_time(e1)/n:.4f} ms/call")
p.close()
