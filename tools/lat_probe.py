"""Single-frame latency breakdown (cfg2): host wall time of the synchronous
host-buffer call vs the device-resident call + stats, the H2D copy alone and
the device time of the frame."""
import math, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, 5.0)
grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0, 0, 0))
p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0))
pose = vm.look_along_x((0, 0, 0))
pa = vm.pose_array([pose])
d = scenes.render(cam, pose, scenes.box_field_boxes(1))
host = torch.from_numpy(d.copy()).pin_memory()
dev = torch.from_numpy(d.copy()).cuda()
def med(f, n=300):
    ts = []
    for _ in range(20): f()
    for _ in range(n):
        t = time.perf_counter(); f(); ts.append(time.perf_counter() - t)
    return np.median(ts) * 1e3, np.percentile(ts, 99) * 1e3
dev_ms = []
def dev_call():
    p.integrate_depth_device(dev.data_ptr(), pa); p.wait_stats()
print("device call + wait_stats  p50/p99 ms %.4f %.4f" % med(dev_call))
print("graph device time ms %.4f" % p.last_frame_ms())
print("host call (H2D + frame + stats) p50/p99 ms %.4f %.4f" % med(lambda: p.integrate_depth_ptr(host.data_ptr(), pa)))
buf = torch.empty_like(dev)
s = torch.cuda.current_stream()
def h2d():
    buf.copy_(host, non_blocking=True); s.synchronize()
print("torch H2D 1.23 MB + sync p50/p99 ms %.4f %.4f" % med(h2d))
print("ctypes no-op (last_frame_ms) p50 ms %.4f" % med(lambda: p.last_frame_ms())[0])
