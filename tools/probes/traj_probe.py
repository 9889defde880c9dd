"""cfg4 trajectory timing as in bench.py (15 calls of 64 frames of the 1000-frame
sweep on device frames), repeated: fresh pipeline per rep (bench form) and a
persistent one. VXM_LIB_NAME selects the library build (A/B)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes, workload as W
dev = torch.device("cuda:0")
c1 = W.CONFIGS["cfg1"]
cam = W.camera(vm, c1)
positions = W.sweep_positions(1000)
poses = [vm.look_along_x(p) for p in positions]
frames = torch.empty((1000, c1["height"], c1["width"]), dtype=torch.float32, device=dev)
vm.render_depth(cam, poses, scenes.corridor_boxes(-60.0, 60.0), out_ptr=frames.data_ptr(), device=0)
torch.cuda.synchronize()
cfg = vm.PipelineConfig(W.grid_for(vm, c1, positions[0]), cam, vox_inf=c1["vox_inf"], depth=c1["depth"])
F = 64
calls = 1000 // F
pa = [vm.pose_array(poses[i * F:(i + 1) * F]) for i in range(calls)]


def run(seq):
    st = torch.cuda.ExternalStream(seq.cuda_stream, device=dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for i in range(calls):
        seq.integrate_depth_device(frames[i * F].data_ptr(), pa[i])
    b.record(st)
    seq.wait_stats()
    return calls * F / (a.elapsed_time(b) / 1000.0)


fresh, pers = [], []
for rep in range(4):
    seq = vm.MappingPipeline(cfg, frames_per_call=F, device=0)
    fresh.append(run(seq))
    seq.close()
seq = vm.MappingPipeline(cfg, frames_per_call=F, device=0)
for rep in range(4):
    pers.append(run(seq))
print("fresh", " ".join(f"{v:.0f}" for v in fresh), "| persistent", " ".join(f"{v:.0f}" for v in pers))
