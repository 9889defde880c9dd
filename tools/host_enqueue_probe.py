"""Host cost of one batched call vs its device time:
(a) pure enqueue: the call issued into an idle context (no ring-slot wait),
timed alone; (b) back to back: per-call submit time when the GPU is busy (it
then includes the wait for a free FrameParams ring slot, i.e. backpressure);
(c) device time per call from CUDA events. The step is device-bound when (a)
is well below (c)."""
import math, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import workload as W

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = W.CONFIGS["cfg2"]
gids = list(range(S))
pipe = W.new_pipeline(vm, c, gids)
cam = W.camera(vm, c)
poses = W.pool_poses(vm)
pool = torch.from_numpy(vm.render_depth(cam, poses, __import__("tests.scenes", fromlist=["x"]).box_field_boxes(1))).cuda()
slots = [pool[torch.tensor([W.frame_of(g, q) for g in gids], device="cuda")].contiguous() for q in range(W.POOL)]
pa = [vm.pose_array([poses[W.frame_of(g, q)] for g in gids]) for q in range(W.POOL)]
for k in range(10):
    pipe.integrate_depth_device(slots[k % W.POOL].data_ptr(), pa[k % W.POOL])
pipe.wait_stats()
idle = []
for k in range(200):
    q = k % W.POOL
    t = time.perf_counter()
    pipe.integrate_depth_device(slots[q].data_ptr(), pa[q])
    idle.append(time.perf_counter() - t)
    pipe.wait_stats()
st = torch.cuda.ExternalStream(pipe.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
busy = []
e0.record(st)
for k in range(400):
    q = k % W.POOL
    t = time.perf_counter()
    pipe.integrate_depth_device(slots[q].data_ptr(), pa[q])
    busy.append(time.perf_counter() - t)
e1.record(st)
pipe.wait_stats()
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) / 400
print(f"S={S}: enqueue into an idle context p50 {np.median(idle)*1e3:.4f} ms (p90 {np.percentile(idle,90)*1e3:.4f}); "
      f"back-to-back submit p50 {np.median(busy)*1e3:.4f} ms (includes ring backpressure); "
      f"device {dev:.4f} ms/call; enqueue/device = {np.median(idle)*1e3/dev:.2f}")
