"""Scratch: host time per vxm_integrate_depth_async call and the e2e rate."""
import math, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
S = 64
cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, 5.0)
grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0, 0, 0))
p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0), n_streams=S)
pose = vm.look_along_x((0, 0, 0))
d = scenes.render(cam, pose, scenes.box_field_boxes(1))
pinned = [torch.from_numpy(np.stack([d] * S)).pin_memory() for _ in range(4)]
poses = [pose] * S
t0 = time.perf_counter(); 
for _ in range(100): p._set_poses(poses)
print("set_poses ms", (time.perf_counter() - t0) * 10)
for k in range(5):
    p.integrate_depth_async(pinned[k % 4].data_ptr(), poses)
p.wait_stats()
for K in (20, 40):
    host = []
    t0 = time.perf_counter()
    for k in range(K):
        t1 = time.perf_counter()
        p.integrate_depth_async(pinned[k % 4].data_ptr(), poses)
        host.append(time.perf_counter() - t1)
    p.wait_stats()
    dt = time.perf_counter() - t0
    print(K, "steps: e2e frames/s %.0f  GB/s %.1f  host ms/call p50 %.3f max %.3f" % (S * K / dt, S * K * d.nbytes / dt / 1e9, 1e3 * np.median(host), 1e3 * max(host)))

# raw H2D while the device-resident pipeline keeps the GPU busy on its own stream
dev = torch.from_numpy(np.stack([d] * S)).cuda()
N = S * d.size
dst = torch.empty(N, dtype=torch.float32, device="cuda")
src = torch.from_numpy(np.stack([d] * S)).reshape(-1).pin_memory()
cs = torch.cuda.Stream()
torch.cuda.synchronize()
for busy in (False, True):
    t0 = time.perf_counter()
    for k in range(16):
        if busy:
            p.integrate_depth_device(dev.data_ptr(), poses)
        with torch.cuda.stream(cs):
            dst.copy_(src, non_blocking=True)
    cs.synchronize()
    dt = time.perf_counter() - t0
    p.wait_stats()
    print("H2D with pipeline busy=%s: %.1f GB/s" % (busy, 16 * N * 4 / dt / 1e9))
