"""Randomised parity sweep (test infrastructure; run under gpurun): random grid
shapes and voxel sizes (odd and even dims_x, rows above and below 128 cells),
camera sizes, vox_inf 0-5, depth limits, general rotations and robot motion
(shifts along every axis, jumps), single streams and batches (desynchronised
branches), compared frame by frame (stats) and grid by grid with the
reference's Sequential pipeline. Prints one summary line per case and a total;
exits non-zero on the first mismatch. A quarter of the cases run the
large-bundle (clear) key format. Usage: python tools/fuzz_parity.py [seconds] [seed]"""
import math, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests.oracle_api import oracle_pipeline

KEYS = ("points_total", "points_outside", "rays_traced", "voxels_freed", "voxels_marked_unknown_traced",
        "voxels_skipped_out_of_bounds", "occupied_count", "freed_count", "shifted", "shift_offset", "origin")


def rotation(rng, tilt):
    yaw, pitch, roll = rng.uniform(-math.pi, math.pi), rng.uniform(-tilt, tilt), rng.uniform(-tilt, tilt)
    cz, sz, cy, sy, cx, sx = math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch), math.cos(roll), math.sin(roll)
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    return vm.look_along_x((0, 0, 0))[0] @ (Rz @ Ry @ Rx)


def aligned_rotation(quarter):
    """look_along_x turned by a multiple of 90 degrees about z (exact 0/1 entries)"""
    c, s = [(1, 0), (0, 1), (-1, 0), (0, -1)][quarter]
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]], dtype=np.float64) @ vm.look_along_x((0, 0, 0))[0]


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else int(time.time()) % 100000
    print("seed", seed, flush=True)
    rng = np.random.default_rng(seed)
    t_end = time.time() + budget
    cases = frames = 0
    while time.time() < t_end:
        # a third of the cases: axis-aligned poses moving by whole voxels through
        # the corridor, so most points lie on voxel faces (near-integer floors,
        # K1's face-heavy warps and per-slot hint)
        aligned = rng.random() < 0.33
        vox = float(rng.choice([0.05, 0.1] if aligned else [0.05, 0.08, 0.1, 0.13, 0.15]))
        ext = rng.uniform([1.5, 1.5, 0.8], [9.0, 6.0, 3.0])
        grid = vm.GridSpec.create_centered(*ext, vox, (0.0, 0.0, 0.0))
        w, h = int(rng.integers(24, 120)), int(rng.integers(18, 90))
        depth_m = float(rng.uniform(2.0, 7.0))
        cam = vm.CameraModel(math.radians(rng.uniform(60, 100)), math.radians(rng.uniform(70, 110)), w, h, depth_m)
        vox_inf = int(rng.integers(0, 6))
        tracer = vm.N.TRACER_PER_PIXEL if rng.random() < 0.15 else vm.N.TRACER_BUNDLED
        cfg = vm.PipelineConfig(grid, cam, vox_inf=vox_inf, depth=depth_m, tracer_mode=tracer)
        S = int(rng.choice([1, 1, 2, 12, 13]))
        n = int(rng.integers(3, 12))
        boxes = scenes.corridor_boxes(-60.0, 60.0) if aligned else scenes.box_field_boxes(int(rng.integers(1, 9)))
        step = rng.integers(-2, 3, 3) * vox if aligned else rng.uniform(-1.5, 1.5, 3) * vox
        tilt = float(rng.uniform(0.0, 0.6))
        quarter = int(rng.integers(0, 4))
        rot = (lambda rng, tilt: aligned_rotation(quarter)) if aligned else rotation
        poses = [[(rot(rng, tilt), np.array([0.1 * s, 0.0, 0.0]) + k * step
                   + (np.array([0.0, 3.0, 0.0]) if k == n // 2 and rng.random() < 0.3 else 0.0))
                  for s in range(S)] for k in range(n)]
        # the large-bundle key format on a quarter of the cases (VXM_FLAG_CLEAR_KEYS)
        kflags = vm.N.FLAG_CLEAR_KEYS if rng.random() < 0.25 else 0
        desc = dict(vox=vox, dims=tuple(grid.dims), cam=(w, h), vox_inf=vox_inf, S=S, n=n, depth=round(depth_m, 3), aligned=aligned,
                    per_pixel=tracer == vm.N.TRACER_PER_PIXEL, clear_keys=bool(kflags))
        print(f"case {cases}: {desc}", flush=True)
        refs = [oracle_pipeline(cfg) for _ in range(S)]
        F = int(rng.choice([1, 1, 1, 2, 5, 33])) if S <= 3 else 1
        if F > 1:
            # multi-frame calls: frames_per_call consecutive frames of each stream
            gpu = vm.MappingPipeline(cfg, n_streams=S, frames_per_call=F, flags=kflags)
            print(f"  frames_per_call {F}", flush=True)
            calls = max(1, n // 2)
            traj = [[(rot(rng, tilt), np.array([0.1 * s, 0.0, 0.0]) + j * step) for j in range(calls * F)]
                    for s in range(S)]
            for c in range(calls):
                ps = [traj[s][c * F + j] for s in range(S) for j in range(F)]
                depth = np.stack([scenes.render(cam, p, boxes) for p in ps])
                st = gpu.integrate_depth(depth, ps)
                for s in range(S):
                    for j in range(F):
                        i = s * F + j
                        sr = refs[s].integrate_depth(depth[i], ps[i])
                        for key in KEYS:
                            if st[i][key] != sr[key]:
                                print(f"MISMATCH case {cases} call {c} stream {s} frame {j} {key}: "
                                      f"{st[i][key]} vs {sr[key]}", flush=True)
                                sys.exit(1)
                frames += S * F
        else:
          gpu = vm.MappingPipeline(cfg, n_streams=S, flags=kflags)
          path = str(rng.choice(["host", "device", "async"]))
          print(f"  path {path}", flush=True)
          keep = []
          for k in range(n):
            depth = np.stack([scenes.render(cam, poses[k][s], boxes) for s in range(S)])
            if path == "host":
                st = gpu.integrate_depth(depth if S > 1 else depth[0], poses[k] if S > 1 else poses[k][0])
                st = st if S > 1 else [st]
            else:
                import torch
                buf = torch.from_numpy(depth).cuda() if path == "device" else torch.from_numpy(depth).pin_memory()
                keep.append(buf)  # (async: the staging copy reads it later)
                if path == "device":
                    gpu.integrate_depth_device(buf.data_ptr(), vm.pose_array(poses[k]))
                else:
                    gpu.integrate_depth_async(buf.data_ptr(), vm.pose_array(poses[k]))
                st = gpu.wait_stats()
            for s in range(S):
                sr = refs[s].integrate_depth(depth[s], poses[k][s])
                for key in KEYS:
                    if st[s][key] != sr[key]:
                        print(f"MISMATCH case {cases} frame {k} stream {s} {key}: {st[s][key]} vs {sr[key]}",
                              dict(vox=vox, dims=tuple(grid.dims), cam=(w, h), vox_inf=vox_inf, S=S), flush=True)
                        sys.exit(1)
            frames += S
        for s in range(S):
            if not np.array_equal(gpu.local_grid(s)[0], refs[s].local_grid()[0]):
                print(f"GRID MISMATCH case {cases} stream {s}", flush=True)
                sys.exit(1)
        gpu.close()
        print(f"case {cases} ok", flush=True)
        cases += 1
    print(f"fuzz parity: {cases} cases, {frames} frames, all bit-exact", flush=True)


if __name__ == "__main__":
    main()
