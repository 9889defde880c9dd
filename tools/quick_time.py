"""Scratch timing of the per-frame graph (device-resident depth) for cfg1/cfg2
batches, plus warm per-stage device times (events between stages, no graph).
QT_CONFIGS="cfg2:64,cfg1:64" selects config:streams pairs."""
import math, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
CFGS = {"cfg1": (0, 6.5), "cfg2": (2, 5.0), "cfg3": (0, 6.5)}
for item in os.environ.get("QT_CONFIGS", "cfg1:1,cfg2:1,cfg2:64,cfg1:64").split(","):
    parts = item.split(":"); name, S = parts[0], int(parts[1]); F = int(parts[2]) if len(parts) > 2 else 1
    vox_inf, dm = CFGS[name]
    if name == "cfg3":  # 1280x720, 0.05 m voxels, 200x200x100
        cam = vm.CameraModel(85 * DEG, 101 * DEG, 1280, 720, dm)
        grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.05, (0, 0, 0))
    else:
        cam = vm.CameraModel(85 * DEG, 101 * DEG, 640, 480, dm)
        grid = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0, 0, 0))
    pose = vm.look_along_x((0, 0, 0))
    d = scenes.render(cam, pose, scenes.box_field_boxes(1))
    if F > 1:  # a moving robot: one voxel per frame along y (cfg4-like)
        poses = [vm.look_along_x((0, 0.1001 * j, 0)) for _ in range(S) for j in range(F)]
    else:
        poses = [pose] * S
    dev = torch.from_numpy(np.stack([d] * (S * F))).cuda()
    xflags = int(os.environ.get("QT_FLAGS", "0"))  # extra context flags (A/B)
    for flags in (xflags, 1 | xflags):
        p = vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=dm), n_streams=S, flags=flags,
                               frames_per_call=F)
        for _ in range(5):
            p.integrate_depth_device(dev.data_ptr(), poses); p.wait_stats()
        ts, st3 = [], []
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if flags & 1:  # whole-stage device times: the four stage-boundary events
            for e in evs:
                e.record(torch.cuda.ExternalStream(p.cuda_stream))
            p.set_stage_events([e.cuda_event for e in evs])
        for k in range(100):
            p.integrate_depth_device(dev.data_ptr(), poses); st = p.wait_stats(); ts.append(p.last_frame_ms())
            if flags & 1:
                st3.append(tuple(evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(3)))
        ts = np.array(ts)
        if not (flags & 1):
            print(f"{name}x{S}x{F} graph p50 ms %.4f p99 %.4f  frames/s %.0f  us/frame %.2f" % (np.median(ts), np.percentile(ts, 99), S * F / np.median(ts) * 1e3, np.median(ts) * 1e3 / (S * F)), flush=True)
        else:
            m = np.median(np.array(st3), axis=0)
            print("   stages (us): populate+dilate %.1f  trace %.1f  merge %.1f   (no-graph total %.1f)" % (m[0], m[1], m[2], np.median(ts) * 1e3), flush=True)
        p.close()
