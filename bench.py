#!/usr/bin/env python3
"""Benchmark of the per-frame voxelization path (arXiv 2112.13169) on B200.

Workload (BASELINE.json configs[1], "cfg2"): 640x480 synthetic depth frames,
0.1 m voxels, 10x10x5 m local grid (100x100x50), vox_inf 2, 5 m depth range,
default FOV 85/101 deg. Every GPU owns S independent sensor streams (default
64, cfg5's batch); one step = one frame for every stream (weak scaling: the
per-GPU work is fixed as N grows; streams shard across ranks with no
collective on the data path).

Frames: a pool of P=16 frames of the reference's box-field scene
(Scene::box_field(1), look_along_x poses y_j = -0.8 + 0.1001 j) rendered on
the host by tests/scenes.py (bit-identical to the reference's render_depth);
stream s at step k consumes pool frame (s + k) mod P, so every stream strafes
~1 voxel per frame and its local grid shifts. The device-side input pool
holds 16 batch slots (1.26 GB), far larger than L2, and consecutive steps
read different slots.

Reported (one JSON line on rank 0):
  value        frames/s of the whole job, device-resident inputs, CUDA events
               on the context's stream around K steps, max over ranks
  e2e          same metric through the C-ABI host-buffer call
               (vxm_integrate_depth: pinned host depth -> H2D -> graph ->
               D2H stats, synchronous per step)
  latency_ms   single-stream per-frame p50/p99: device (events) and e2e (wall)
  roofline     dominant kernel (K3 trace_bundle), see DESIGN.md §Roofline
  cpu_baseline the reference's own CPU code (oracle/_ref/ref_bench, built
               from /root/reference sources) on this box's cores
--impl reference runs only the reference CPU implementation (all host
threads) on the same workload and prints its line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

DEG = math.pi / 180.0
CFG = dict(name="cfg2", width=640, height=480, vox=0.1, grid=(10.0, 10.0, 5.0), vox_inf=2, depth=5.0)
POOL = 16
Y0 = -0.8
MEASURED_PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--streams", type=int, default=64, help="sensor streams per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--latency-frames", type=int, default=300)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    from paper_2112_13169_b200 import multi
    return multi.env()


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def ref_bench_cmd(streams, steps, warmup, threads):
    exe = ROOT / "oracle" / "_ref" / "ref_bench"
    if not exe.exists():
        return None
    c = CFG
    return [str(exe), "--width", str(c["width"]), "--height", str(c["height"]), "--vox", str(c["vox"]),
            "--gx", str(c["grid"][0]), "--gy", str(c["grid"][1]), "--gz", str(c["grid"][2]),
            "--depth", str(c["depth"]), "--vox-inf", str(c["vox_inf"]), "--streams", str(streams),
            "--steps", str(steps), "--warmup", str(warmup), "--pool", str(POOL), "--y0", str(Y0),
            "--threads", str(threads)]


def run_ref(streams, steps, warmup, threads):
    cmd = ref_bench_cmd(streams, steps, warmup, threads)
    if cmd is None:
        return None
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    if out.returncode != 0:
        return None
    return json.loads(out.stdout.strip().splitlines()[-1])


def config_dict(streams, n):
    c = CFG
    return {"workload": f"{c['name']}: {c['width']}x{c['height']} synthetic depth, {c['vox']} m voxels, "
                        f"{int(c['grid'][0] / c['vox'])}x{int(c['grid'][1] / c['vox'])}x{int(c['grid'][2] / c['vox'])} grid, "
                        f"vox_inf {c['vox_inf']}, {c['depth']} m depth; {streams} streams per GPU",
            "frame_shape": [c["height"], c["width"]], "vox_size": c["vox"], "grid_dims": [100, 100, 50],
            "vox_inf": c["vox_inf"], "depth_m": c["depth"], "streams_per_gpu": streams, "n_gpus": n,
            "streams_total": streams * n, "l2": "inputs larger than L2 (16 x S frame slots, 1.26 GB at S=64)",
            "parallelism": f"{n} GPU(s) x {streams} independent streams, no collective"}


# --------------------------------------------------------------------------- reference arm

def reference_arm(args, world, rank):
    if rank != 0:
        return
    cores = host_cores()
    r = run_ref(args.streams, args.steps, args.warmup, cores)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_bench not built"}))
        return
    line = {"metric": "frames_per_s", "value": round(r["frames_per_s"], 3), "unit": "frames/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 * r["seconds"] / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.streams, 1),
            "latency_ms": {"p50": r["p50_ms"], "p99": r["p99_ms"], "note": "per frame, one stream per thread"},
            "cpu_baseline": {"value": round(r["frames_per_s"], 3), "unit": "frames/s", "cores": r["threads"],
                             "kind": "reference",
                             "sample": f"{r['frames']} frames ({args.streams} streams x {args.steps} steps), "
                                       f"Sequential MappingPipeline per stream, {cpu_model()}"},
            "e2e": {"value": round(r["frames_per_s"], 3), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm

class ClockSampler:
    """SM clock and clock-event reasons polled through NVML (~1 ms period)
    by a thread while the timed region runs (an nvidia-smi subprocess cannot
    sample a region of a few milliseconds)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                             pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:
                        pass
                    time.sleep(0.001)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
            time.sleep(0.005)  # at least one sample before the region starts
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return None
        reasons = sorted(n for n, bit in self.REASONS.items() if any(r & bit for _, r in self.samples))
        return {"sm_mhz": statistics.median(c for c, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


def hbm_peak():
    if MEASURED_PEAKS.exists():
        try:
            d = json.loads(MEASURED_PEAKS.read_text())
            for k in ("hbm_gbs", "hbm_GBps", "hbm"):
                if k in d:
                    return float(d[k]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


def profiled_traffic():
    """dram bytes per trace launch (and the pipe utilisation) from the
    committed ncu --set full capture."""
    f = ROOT / "profiles" / "trace_traffic.json"
    if f.exists():
        try:
            d = json.loads(f.read_text())
            return d.get("dram_bytes_per_launch"), d
        except Exception:
            pass
    return None, None


def our_arm(args, world, rank, local):
    import numpy as np
    import torch

    from paper_2112_13169_b200 import _native as N
    from paper_2112_13169_b200 import multi
    from paper_2112_13169_b200 import voxmap as vm
    from tests import scenes

    dist = world > 1
    if dist:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = CFG
    S, K, WU = args.streams, args.steps, max(3, args.warmup)
    cam = vm.CameraModel(85 * DEG, 101 * DEG, c["width"], c["height"], c["depth"])
    boxes = scenes.box_field_boxes(1)
    poses = [vm.look_along_x((0.0, Y0 + 0.1001 * j, 0.0)) for j in range(POOL)]
    # the frame pool is rendered on the GPU (vxm_render_depth, bit-identical to
    # the reference's sim::render_depth); frame 0 is checked against the host
    pool = vm.render_depth(cam, poses, boxes, device=local)  # (P, H, W)
    assert np.array_equal(pool[0], scenes.render(cam, poses[0], boxes))
    npix = c["width"] * c["height"]

    # this rank's streams (global ids); slot q holds, for every stream g,
    # pool frame (g + q) mod P
    gids = list(multi.stream_range(S, rank))
    pool_dev = torch.from_numpy(pool).to(dev)
    slots = torch.empty((POOL, S, c["height"], c["width"]), dtype=torch.float32, device=dev)
    for q in range(POOL):
        idx = torch.tensor([(g + q) % POOL for g in gids], device=dev)
        slots[q] = pool_dev[idx]
    torch.cuda.synchronize()

    # step k's poses, packed once per pool phase (vxm_pose layout) so the
    # timed loops pass one array per call instead of marshalling S poses
    pose_phase = [vm.pose_array([poses[(g + q) % POOL] for g in gids]) for q in range(POOL)]

    def step_poses(k):
        return pose_phase[k % POOL]

    def new_pipeline(streams, flags=0):
        g0 = vm.GridSpec.create_centered(*c["grid"], c["vox"], poses[0][1])
        p = vm.MappingPipeline(vm.PipelineConfig(g0, cam, vox_inf=c["vox_inf"], depth=c["depth"]),
                               n_streams=streams, device=local, flags=flags)
        for s in range(streams):
            p.set_origin(vm.GridSpec.create_centered(*c["grid"], c["vox"], poses[gids[s] % POOL][1]).origin, s)
        return p

    # ---- device-resident throughput (value): the default batch graph, whose
    # branches overlap the stages of different stream shares
    pipe = new_pipeline(S)
    branches = pipe.graph_branches
    pipe_dims = tuple(vm.GridSpec.create_centered(*c["grid"], c["vox"], poses[0][1]).dims)
    stream = torch.cuda.ExternalStream(pipe.cuda_stream, device=dev)
    for k in range(WU):
        pipe.integrate_depth_device(slots[k % POOL].data_ptr(), step_poses(k))
    pipe.wait_stats()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        start.record(stream)
        for k in range(K):
            pipe.integrate_depth_device(slots[(WU + k) % POOL].data_ptr(), step_poses(WU + k))
        end.record(stream)
        stats = pipe.wait_stats()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    ms = multi.max_over_ranks(ms, dev)
    value = multi.job_throughput(S * K, world, ms / 1000.0)
    # K1 populate, K2 dilation when vox_inf > 0 (one fused tile kernel when dims_x % 4 == 0, else K2a rows +
    # K2b tiles), K3 trace, K4 merge, K5 publish, per branch
    k2 = 0 if c["vox_inf"] == 0 else (1 if pipe_dims[0] % 4 == 0 else 2)
    kernels_per_step = (4 + k2) * branches

    # ---- per-kernel device times (the roofline's K3 duration): the same
    # steps as ONE graph branch, stage-boundary events recorded inside the
    # graph on the launching stream, so each stage is timed alone
    kpipe = new_pipeline(S, flags=N.FLAG_SINGLE_BRANCH | N.FLAG_STAGE_EVENTS)
    kstream = torch.cuda.ExternalStream(kpipe.cuda_stream, device=dev)
    for k in range(WU):
        kpipe.integrate_depth_device(slots[k % POOL].data_ptr(), step_poses(k))
    kpipe.wait_stats()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    for e4 in ev:
        for e in e4:
            e.record(kstream)  # materialise the handles
    kstart, kend = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    kstart.record(kstream)
    for k in range(K):
        kpipe.set_stage_events([e.cuda_event for e in ev[k]])
        kpipe.integrate_depth_device(slots[(WU + k) % POOL].data_ptr(), step_poses(WU + k))
    kend.record(kstream)
    kpipe.wait_stats()
    torch.cuda.synchronize()
    kpipe.set_stage_events(None)
    single_branch_ms = kstart.elapsed_time(kend) / K
    trace_ms = [e4[1].elapsed_time(e4[2]) for e4 in ev]
    stage_ms = {"populate_dilate": statistics.mean(e4[0].elapsed_time(e4[1]) for e4 in ev),
                "trace": statistics.mean(trace_ms),
                "merge_shift_count": statistics.mean(e4[2].elapsed_time(e4[3]) for e4 in ev)}
    kpipe.close()

    # ---- end to end through the C-ABI host-buffer call
    pinned = torch.empty((POOL, S, c["height"], c["width"]), dtype=torch.float32).pin_memory()
    pool_cpu = torch.from_numpy(pool)
    for q in range(POOL):
        pinned[q].copy_(pool_cpu[torch.tensor([(g + q) % POOL for g in gids])])
    e2e_pipe = new_pipeline(S)
    for k in range(WU):
        e2e_pipe.integrate_depth_async(pinned[k % POOL].data_ptr(), step_poses(k))
    e2e_pipe.wait_stats()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    # vxm_integrate_depth_async: pinned host frames -> H2D on the copy stream
    # (double buffered) -> frame graph -> D2H of the counters; the timed region
    # ends when the last frame's stats are on the host.
    t0 = time.perf_counter()
    for k in range(K):
        e2e_pipe.integrate_depth_async(pinned[(WU + k) % POOL].data_ptr(), step_poses(WU + k))
    e2e_stats = e2e_pipe.wait_stats()
    e2e_s = time.perf_counter() - t0
    assert e2e_stats[0]["occupied_count"] == stats[0]["occupied_count"]  # same frames, same result
    e2e_s = multi.max_over_ranks(e2e_s, dev)
    e2e_value = multi.job_throughput(S * K, world, e2e_s)
    h2d = S * npix * 4 + S * 160  # depth frames + per-stream FrameParams
    d2h = S * 96                  # per-stream counters + stage stamps (vxm::kCountersHostBytes)
    e2e_pipe.close()

    # ---- single-stream latency
    lat = new_pipeline(1)
    one = torch.empty((1, c["height"], c["width"]), dtype=torch.float32).pin_memory()
    one_pose = [vm.pose_array([poses[j]]) for j in range(POOL)]  # vxm_pose layout, packed once
    dev_lat, e2e_lat = [], []
    for k in range(args.latency_frames + 10):
        j = k % POOL
        lat.integrate_depth_device(pool_dev[j].data_ptr(), one_pose[j])
        lat.wait_stats()
        if k >= 10:
            dev_lat.append(lat.last_frame_ms())
    lat.close()
    lat = new_pipeline(1)
    for k in range(args.latency_frames + 10):
        j = k % POOL
        one[0].copy_(torch.from_numpy(pool[j]))
        t1 = time.perf_counter()
        lat.integrate_depth_ptr(one.data_ptr(), one_pose[j])
        if k >= 10:
            e2e_lat.append((time.perf_counter() - t1) * 1000.0)
    lat.close()

    # ---- one moving robot (cfg4-style trajectory): F consecutive frames per
    # call (vxm_create_multi), device-resident frames; the sequential
    # single-frame rate of the same trajectory is latency_ms above
    F = 64
    g0 = vm.GridSpec.create_centered(*c["grid"], c["vox"], poses[0][1])
    traj = vm.MappingPipeline(vm.PipelineConfig(g0, cam, vox_inf=c["vox_inf"], depth=c["depth"]),
                              frames_per_call=F, device=local)
    order = [j % POOL for j in range(F)]
    traj_dev = pool_dev[torch.tensor(order, device=dev)].contiguous()
    traj_poses = vm.pose_array([poses[j] for j in order])
    tstream = torch.cuda.ExternalStream(traj.cuda_stream, device=dev)
    for _ in range(3):
        traj.integrate_depth_device(traj_dev.data_ptr(), traj_poses)
    traj.wait_stats()
    calls = max(10, K // 2)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_start.record(tstream)
    for _ in range(calls):
        traj.integrate_depth_device(traj_dev.data_ptr(), traj_poses)
    t_end.record(tstream)
    traj_stats = traj.wait_stats()
    torch.cuda.synchronize()
    traj_ms = t_start.elapsed_time(t_end)
    traj.close()
    trajectory = {"frames_per_call": F, "calls": calls, "frames_per_s": round(F * calls / (traj_ms / 1000.0), 1),
                  "us_per_frame": round(traj_ms * 1000.0 / (F * calls), 3),
                  "shifted_frames_per_call": int(sum(st["shifted"] for st in traj_stats)),
                  "note": "one stream, 64 consecutive frames per call (chain-folded merge); "
                          "device-resident frames, CUDA events"}

    def pct(v, q):
        v = sorted(v)
        pos = q * (len(v) - 1)
        lo = int(pos)
        hi = min(lo + 1, len(v) - 1)
        return v[lo] + (pos - lo) * (v[hi] - v[lo])

    # ---- roofline of the dominant kernel (K3): SURVEY §8d algorithmic bytes
    # per frame (4*W*H + 4*N) x the S frames one launch processes / its time
    bytes_per_frame = 4 * npix + 4 * 500000
    trace_avg_s = statistics.mean(trace_ms) / 1000.0
    achieved = bytes_per_frame * S / trace_avg_s / 1e9
    peak, peak_kind = hbm_peak()
    traffic, prof = profiled_traffic()

    line = {"metric": "frames_per_s", "value": round(value, 1), "unit": "frames/s", "n_gpus": world,
            "steps": K, "warmup": WU, "ms_per_step": round(ms / K, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(S, world),
            "e2e": {"value": round(e2e_value, 1), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "latency_ms": {"p50": round(pct(dev_lat, 0.5), 4), "p99": round(pct(dev_lat, 0.99), 4),
                           "e2e_p50": round(pct(e2e_lat, 0.5), 4), "e2e_p99": round(pct(e2e_lat, 0.99), 4),
                           "frames": len(dev_lat), "note": "one stream, one frame at a time"},
            "stage_ms_per_step": {k: round(v, 4) for k, v in stage_ms.items()},
            "graph_branches": branches,
            "single_branch_ms_per_step": round(single_branch_ms, 4),
            "trajectory": trajectory,
            "roofline": {"bound": "hbm", "kernel": "trace_bundle_kernel", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": peak_kind,
                         "bytes_per_launch": bytes_per_frame * S,
                         # K3 is not HBM-bound: ncu shows its ALU pipe as the binding unit
                         "binding_pipe": None if not prof else {
                             "pipe": "alu", "pct_of_peak": prof.get("alu_pipe_pct_of_peak"),
                             "issue_active_pct": prof.get("issue_active_pct"),
                             "source": f"profiles/{prof.get('tag')}_kernels.md (ncu --set full)"}},
            "gpu_launches": kernels_per_step * K,
            "hbm_gbs_pipeline": round(bytes_per_frame * value / world / 1e9, 1),
            "checks": {"occupied_count_s0": stats[0]["occupied_count"], "freed_count_s0": stats[0]["freed_count"]}}
    cl = clocks.summary()
    if cl:
        line["clocks"] = cl
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        r = run_ref(64, 8, 1, cores)
        if r:
            line["cpu_baseline"] = {"value": round(r["frames_per_s"], 3), "unit": "frames/s", "cores": r["threads"],
                                    "kind": "reference",
                                    "sample": f"{r['frames']} frames (64 streams x 8 steps, same pool/rule), "
                                              f"Sequential MappingPipeline per stream, {cpu_model()}",
                                    "latency_ms_p50": r["p50_ms"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    pipe.close()
    if dist:
        tdist.barrier()
        tdist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    our_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
