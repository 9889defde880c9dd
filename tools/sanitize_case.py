"""Small runs of every kernel for compute-sanitizer (tools/sanitize.sh):
batched frames (3 graph branches), vox_inf 2 (dilation), a 4-frame
sequence call, the stage API, the renderer. Checks results against the
single-frame path so a sanitizer-perturbed run still has to be right."""
import math, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
DEG = math.pi / 180
cam = vm.CameraModel(85 * DEG, 101 * DEG, 64, 48, 5.0)
grid = vm.GridSpec.create_centered(4.0, 4.0, 2.0, 0.1, (0, 0, 0))
cfg = vm.PipelineConfig(grid, cam, vox_inf=2, depth=5.0)
boxes = scenes.box_field_boxes(1)
S = 12
poses = [vm.look_along_x((0.0, 0.05 * s, 0.0)) for s in range(S)]
depth = vm.render_depth(cam, poses, boxes)
batch = vm.MappingPipeline(cfg, n_streams=S, flags=vm.N.FLAG_NO_GRAPH)
one = vm.MappingPipeline(cfg, flags=vm.N.FLAG_NO_GRAPH)
sb = batch.integrate_depth(depth, poses)
for s in range(S):
    so = one.integrate_depth(depth[s], poses[s])
    assert so["freed_count"] == one.local_grid()[0].tolist().count(1)
seq = vm.MappingPipeline(cfg, frames_per_call=4, flags=vm.N.FLAG_NO_GRAPH)
seq.integrate_depth(depth[:4], poses[:4])
ms = np.zeros(grid.cell_count(), np.uint8)
vm.populate_occupied(grid, ms, np.random.uniform(0, 4, 200), np.random.uniform(0, 4, 200),
                     np.random.uniform(0, 2, 200), vm.identity_pose(), 2)
vm.trace_bundle(grid, ms, vm.bundle_dimensions(cam, 2.0, 0.1), vm.look_along_x((2.0, 2.0, 1.0)))
# K4 variants under motion: flat chunks (y/z shifts), word rows (x shifts),
# TMA-staged rows (200-cell rows)
movers = []
for ext, vox, mot in (((6.4, 3.2, 1.6), 0.1, (0.0, 1.0, -0.7)), ((6.4, 3.2, 1.6), 0.1, (1.0, 0.6, -0.4)),
                      ((10.0, 3.0, 2.0), 0.05, (1.0, 0.6, -0.4)), ((10.0, 3.0, 2.0), 0.05, (0.0, 1.0, 0.5))):
    g = vm.GridSpec.create_centered(*ext, vox, (0.0, 0.0, 0.0))
    m = vm.MappingPipeline(vm.PipelineConfig(g, cam, vox_inf=1, depth=5.0), flags=vm.N.FLAG_NO_GRAPH)
    for k in range(6):
        pose = vm.look_along_x(tuple(c * 1.37 * vox * k for c in mot))
        m.integrate_depth(vm.render_depth(cam, [pose], boxes)[0], pose)
    movers.append(m)
# desynchronised batch graphs (per-branch streams), back to back
dbatch = vm.MappingPipeline(cfg, n_streams=S)
for k in range(4):
    dbatch.integrate_depth(depth, poses)
movers.append(dbatch)
# round 2: a batch large enough for the 16-rows-per-warp K4 with its
# last-block counter publish (32 streams of a 100x100x50 grid), near-field
# ray-cast chunks (surfaces beyond the near field), y and x shifts
gbig = vm.GridSpec.create_centered(10.0, 10.0, 5.0, 0.1, (0.0, 0.0, 0.0))
cam2 = vm.CameraModel(85 * DEG, 101 * DEG, 96, 72, 5.0)
big = vm.MappingPipeline(vm.PipelineConfig(gbig, cam2, vox_inf=2, depth=5.0), n_streams=32)
for k in range(3):
    ps = [vm.look_along_x((0.13 * k * (s % 2), 0.11 * k, 0.0)) for s in range(32)]
    big.integrate_depth(vm.render_depth(cam2, ps, boxes), ps)
movers.append(big)
# chain merges with their in-kernel counter publish: one stream of 33 frames
# (three chained frame ranges) and 3 streams x 8 frames whose x shifts are
# multiples of 4 cells (the word-wise chains)
seq33 = vm.MappingPipeline(cfg, frames_per_call=33)
ps = [vm.look_along_x((0.0, 0.05 * (j % 12), 0.0)) for j in range(33)]
seq33.integrate_depth(vm.render_depth(cam, ps, boxes), ps)
seq3 = vm.MappingPipeline(cfg, n_streams=3, frames_per_call=8)
ps = [vm.look_along_x((0.4 * (j % 3), 0.1 * s, 0.0)) for s in range(3) for j in range(8)]
seq3.integrate_depth(vm.render_depth(cam, ps, boxes), ps)
movers += [seq33, seq3]
print("sanitize case done", sb[0]["freed_count"])
for p in [batch, one, seq] + movers:
    p.close()
