"""The benchmark workload (synthetic inputs, host side): shared by bench.py and
tests/test_gpu_bench_parity.py so the parity test runs exactly what the
bench times.

BASELINE.json configs:
  cfg1  640x480, 0.1 m voxels, 100x100x50 grid, vox_inf 0, 6.5 m depth
  cfg2  640x480, 0.1 m voxels, 100x100x50 grid, vox_inf 2, 5 m depth
  cfg3  1280x720, 0.05 m voxels, 200x200x100 grid, vox_inf 0, 6.5 m depth
  cfg4  1000-frame sweep_trajectory((0,-50,0),(0,50,0),1000) on cfg1 frames
        (proj/src/sim/trajectory.cpp:15-25) through the corridor scene
  cfg5  64 independent cfg2 streams, sharded over 1/2/4/8 GPUs

Frame rule of the batched configs (also oracle/ref_bench.cpp): a pool of
P = 16 look_along_x poses y_j = Y0 + 0.1001 j over Scene::box_field(1);
stream g at step k consumes pool frame (g + k) mod P, so each stream strafes
about one voxel per frame (its local grid shifts) and jumps back 1.5 m when
the pool wraps. Stream g's grid starts centred on pool pose g mod P.
"""
from __future__ import annotations

import math

DEG = math.pi / 180.0
POOL = 16
Y0 = -0.8

CONFIGS = {
    "cfg1": dict(name="cfg1", width=640, height=480, vox=0.1, grid=(10.0, 10.0, 5.0), vox_inf=0, depth=6.5),
    "cfg2": dict(name="cfg2", width=640, height=480, vox=0.1, grid=(10.0, 10.0, 5.0), vox_inf=2, depth=5.0),
    "cfg3": dict(name="cfg3", width=1280, height=720, vox=0.05, grid=(10.0, 10.0, 5.0), vox_inf=0, depth=6.5),
}


def pool_y(j: int) -> float:
    return Y0 + 0.1001 * j


def camera(vm, c):
    return vm.CameraModel(85 * DEG, 101 * DEG, c["width"], c["height"], c["depth"])


def pool_poses(vm):
    return [vm.look_along_x((0.0, pool_y(j), 0.0)) for j in range(POOL)]


def grid_for(vm, c, center):
    return vm.GridSpec.create_centered(*c["grid"], c["vox"], center)


def pipeline_config(vm, c):
    poses = pool_poses(vm)
    return vm.PipelineConfig(grid_for(vm, c, poses[0][1]), camera(vm, c), vox_inf=c["vox_inf"], depth=c["depth"])


def dims(vm, c):
    return tuple(grid_for(vm, c, (0.0, 0.0, 0.0)).dims)


def cells(vm, c) -> int:
    d = dims(vm, c)
    return d[0] * d[1] * d[2]


def frame_of(g: int, k: int) -> int:
    """pool frame of global stream g at step k"""
    return (g + k) % POOL


def new_pipeline(vm, c, gids, device=0, flags=0):
    """A batched pipeline over global streams `gids`, each grid centred on its
    stream's first pose (pipeline.hpp:63), as oracle/ref_bench.cpp sets up."""
    poses = pool_poses(vm)
    p = vm.MappingPipeline(pipeline_config(vm, c), n_streams=len(gids), device=device, flags=flags)
    for s, g in enumerate(gids):
        p.set_origin(grid_for(vm, c, poses[g % POOL][1]).origin, s)
    return p


def sweep_positions(frames=1000, start=(0.0, -50.0, 0.0), end=(0.0, 50.0, 0.0)):
    """sim::sweep_trajectory (proj/src/sim/trajectory.cpp:15-25): start +
    s * (end - start), s = i / (frames - 1), element-wise in that order."""
    out = []
    for i in range(frames):
        s = 0.0 if frames == 1 else i / (frames - 1)
        out.append(tuple(start[a] + s * (end[a] - start[a]) for a in range(3)))
    return out
