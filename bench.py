#!/usr/bin/env python3
"""Benchmark of the per-frame voxelization path (arXiv 2112.13169) on B200.

Headline workload (BASELINE.json configs[1], "cfg2", batched as configs[4]
"cfg5"): 640x480 synthetic depth frames, 0.1 m voxels, 10x10x5 m local grid
(100x100x50), vox_inf 2, 5 m depth range, default FOV 85/101 deg; S
independent sensor streams per GPU (default 64); one step = one frame for
every stream. --scaling weak (default): S streams per GPU, the per-GPU work
is fixed as N grows; --scaling strong: S streams in total, S/N per GPU (cfg5
as written). Streams shard across ranks with no collective on the data path.

Frames (tests/workload.py, shared with the parity tests): a pool of P=16
frames of the reference's box-field scene (Scene::box_field(1), look_along_x
poses y_j = -0.8 + 0.1001 j) rendered on the GPU by vxm_render_depth
(bit-identical to the reference's render_depth; frame 0 is checked against
the host renderer); stream g at step k consumes pool frame (g + k) mod P, so
every stream strafes ~1 voxel per frame, its local grid shifts, and it jumps
back 1.5 m when the pool wraps. The device-side input pool holds 16 batch
slots (1.26 GB at S=64), far larger than L2, and consecutive steps read
different slots.

Reported (one JSON line on rank 0):
  value        frames/s of the whole job, device-resident inputs, CUDA events
               on the context's stream around K back-to-back steps, max over
               ranks
  e2e          the same through the C-ABI asynchronous host-buffer call
               (vxm_integrate_depth_async: pinned host frames -> H2D on a
               copy stream, double buffered -> frame graphs -> counters
               written into host-mapped memory), wall clock until the last
               step's stats are on the host
  parity       the timed runs' final grids, origins and last-step stats of
               every stream against the reference's own code run on the same
               frames (oracle/_ref/ref_bench), for cfg2 and the other configs
  latency_ms   one stream, one frame at a time, >= 1000 frames: device time
               (events) and e2e wall time (pinned host frame -> stats)
  configs      cfg1 x 64 and cfg3 x 16 batches, the cfg4 1000-frame sweep
  roofline     the dominant kernel (K3 trace_bundle), DESIGN.md §8
  cpu_baseline the reference's own CPU code (oracle/_ref/ref_bench, built
               from /root/reference sources) on this box's cores: batch
               throughput and single-frame latency (Sequential on 1 core,
               DataParallel on all cores)
--impl reference runs only the reference CPU implementation (all host
threads) on the same workload and prints its line.
Without WORLD_SIZE in the environment, --gpus N > 1 relaunches this script
under torch.distributed.run with N ranks (one per GPU; ranks share GPUs when
fewer are visible, with gloo for the barrier and the max).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from tests import workload as W  # noqa: E402  (synthetic inputs, host side)

MEASURED_PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
HEADLINE = "cfg2"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--streams", type=int, default=64,
                    help="sensor streams per GPU (weak) or in total (strong)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--latency-frames", type=int, default=1000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="headline only (no other configs / latency)")
    ap.add_argument("--plumbing-only", action="store_true",
                    help="distributed launch + timing plumbing without GPU work (CPU test of the N>1 path)")
    return ap.parse_args()


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


def streams_per_rank(args, world):
    if args.scaling == "strong":
        if args.streams % world:
            raise SystemExit(f"--scaling strong needs --streams ({args.streams}) divisible by the GPU count ({world})")
        return args.streams // world
    return args.streams


def config_dict(c, S, world, scaling):
    import paper_2112_13169_b200.voxmap as vm
    d = W.dims(vm, c)
    return {"workload": f"{c['name']}: {c['width']}x{c['height']} synthetic depth, {c['vox']} m voxels, "
                        f"{d[0]}x{d[1]}x{d[2]} grid, vox_inf {c['vox_inf']}, {c['depth']} m depth; "
                        f"{S} streams per GPU",
            "frame_shape": [c["height"], c["width"]], "vox_size": c["vox"], "grid_dims": list(d),
            "vox_inf": c["vox_inf"], "depth_m": c["depth"], "streams_per_gpu": S, "n_gpus": world,
            "streams_total": S * world, "scaling": scaling,
            "l2": f"inputs larger than L2 ({W.POOL} x S frame slots, "
                  f"{W.POOL * S * c['width'] * c['height'] * 4 / 1e9:.2f} GB per GPU)",
            "parallelism": f"{world} GPU(s) x {S} independent streams, no collective"}


# --------------------------------------------------------------------------- launch

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(n):
    """bench.py --gpus N without a torchrun environment: one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def init_dist(world, local):
    """process group for the barrier and the max over ranks: NCCL when every
    rank has its own GPU, else gloo (ranks sharing a GPU, or CPU plumbing)."""
    import torch
    import torch.distributed as tdist

    if world <= 1:
        return None
    ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    backend = "nccl" if ngpu >= world else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(local)
    tdist.init_process_group(backend)
    return backend


# --------------------------------------------------------------------------- reference arm

def reference_arm(args, world, rank):
    if rank != 0:
        return  # rank 0 alone times the host CPU reference
    from oracle import ref_bench

    S = streams_per_rank(args, world)
    c = W.CONFIGS[HEADLINE]
    cores = host_cores()
    if not ref_bench.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_bench not built"}))
        return
    # the whole job's streams (S per GPU x N GPUs) on the host's cores
    r = ref_bench.run(c, S * world, args.steps, args.warmup, cores, pool=W.POOL, y0=W.Y0)
    line = {"metric": "frames_per_s", "value": round(r["frames_per_s"], 3), "unit": "frames/s",
            "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 * r["seconds"] / args.steps, 3), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(c, S, world, args.scaling),
            "latency_ms": {"p50": r["p50_ms"], "p99": r["p99_ms"], "note": "per frame, one stream per thread"},
            "cpu_baseline": {"value": round(r["frames_per_s"], 3), "unit": "frames/s", "cores": r["threads"],
                             "kind": "reference",
                             "sample": f"{r['frames']} frames ({S * world} streams x {args.steps} steps), "
                                       f"Sequential MappingPipeline per stream, {cpu_model()}"},
            "e2e": {"value": round(r["frames_per_s"], 3), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- plumbing-only arm (CPU)

def plumbing_arm(args, world, rank, local):
    """The N>1 launch and timing plumbing without GPU work: rank/world, the
    stream shard of each rank, a timed region (rank r sleeps r*10 ms) and the
    max over ranks. tests/test_distributed_gloo.py runs it on CPU."""
    import torch
    import torch.distributed as tdist

    from paper_2112_13169_b200 import multi

    backend = init_dist(world, local)
    S = streams_per_rank(args, world)
    gids = list(multi.stream_range(S, rank))
    if backend:
        tdist.barrier()
    t0 = time.perf_counter()
    time.sleep(0.01 * rank)
    el = time.perf_counter() - t0
    el = multi.max_over_ranks(el)
    owned = [None] * world
    if backend:
        tdist.all_gather_object(owned, [gids[0], gids[-1]])
    else:
        owned = [[gids[0], gids[-1]]]
    if rank == 0:
        print(json.dumps({"metric": "frames_per_s", "value": round(multi.job_throughput(S * args.steps, world, el), 1),
                          "n_gpus": world, "backend": backend, "scaling": args.scaling,
                          "streams_per_rank": S, "owned": owned, "max_seconds": el,
                          "config": {"streams_per_gpu": S, "n_gpus": world, "streams_total": S * world}}),
              flush=True)
    if backend:
        tdist.barrier()
        tdist.destroy_process_group()
    del torch


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


def step_instructions():
    """warp instructions of one batched cfg2 step (64 frames) from the committed
    ncu capture (tools/summarize_profiles.py -> profiles/step_instructions.json)"""
    f = ROOT / "profiles" / "step_instructions.json"
    if f.exists():
        try:
            return json.loads(f.read_text())
        except Exception:
            pass
    return None


def pct(v, q):
    v = sorted(v)
    pos = q * (len(v) - 1)
    lo = int(pos)
    hi = min(lo + 1, len(v) - 1)
    return v[lo] + (pos - lo) * (v[hi] - v[lo])


class Workload:
    """One config's device-resident slots, pinned copies and packed poses for
    this rank's streams (tests/workload.py frame rule)."""

    def __init__(self, vm, torch, dev, c, gids, pinned=False):
        self.c, self.gids, self.dev = c, gids, dev
        S = len(gids)
        cam = W.camera(vm, c)
        self.poses = W.pool_poses(vm)
        pool = vm.render_depth(cam, self.poses, _boxes(), device=dev.index or 0)  # (P, H, W), bit-identical
        self.pool_host = pool
        pool_dev = torch.from_numpy(pool).to(dev)
        self.pool_dev = pool_dev
        self.slots = torch.empty((W.POOL, S, c["height"], c["width"]), dtype=torch.float32, device=dev)
        for q in range(W.POOL):
            self.slots[q] = pool_dev[torch.tensor([W.frame_of(g, q) for g in gids], device=dev)]
        self.pinned = None
        if pinned:
            self.pinned = torch.empty((W.POOL, S, c["height"], c["width"]), dtype=torch.float32).pin_memory()
            self.pinned.copy_(self.slots.cpu())
        # step k's poses, packed once per pool phase (vxm_pose layout)
        self.pose_phase = [vm.pose_array([self.poses[W.frame_of(g, q)] for g in gids]) for q in range(W.POOL)]
        torch.cuda.synchronize()

    def step(self, k):
        return self.slots[k % W.POOL].data_ptr(), self.pose_phase[k % W.POOL]

    def host_step(self, k):
        return self.pinned[k % W.POOL].data_ptr(), self.pose_phase[k % W.POOL]


def _boxes():
    from tests import scenes
    return scenes.box_field_boxes(1)


def final_state(vm, pipe, S):
    import numpy as np
    grids, origins = [], []
    for s in range(S):
        g, o = pipe.local_grid(s)
        grids.append(g)
        origins.append(o)
    return np.stack(grids), np.stack(origins)


def compare_with_reference(ref, got_grids, got_origins, got_last):
    """parity of a timed run's end state with ref_bench's dumps"""
    import numpy as np

    from oracle import ref_bench
    last = np.array([ref_bench.stats_row(st) for st in got_last])
    bad_grids = [int(s) for s in range(len(got_grids)) if not np.array_equal(got_grids[s], ref["grids"][s])]
    ok = (not bad_grids and np.array_equal(got_origins, ref["origins"])
          and np.array_equal(last, ref["stats"][-1]))
    return ok, bad_grids


def timed_batch(vm, torch, dev, wl, S, K, WU, flags=0, clocks=None, dist_barrier=None):
    """K back-to-back device-resident steps after WU warm-up steps; returns
    (ms over K steps, pipeline, last stats)."""
    from paper_2112_13169_b200 import multi
    pipe = W.new_pipeline(vm, wl.c, wl.gids, device=dev.index or 0, flags=flags)
    stream = torch.cuda.ExternalStream(pipe.cuda_stream, device=dev)
    for k in range(WU):
        pipe.integrate_depth_device(*wl.step(k))
    pipe.wait_stats()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist_barrier:
        dist_barrier()
    torch.cuda.synchronize()
    ctx = clocks if clocks is not None else _Null()
    with ctx:
        start.record(stream)
        for k in range(K):
            pipe.integrate_depth_device(*wl.step(WU + k))
        end.record(stream)
        stats = pipe.wait_stats()
        torch.cuda.synchronize()
    ms = multi.max_over_ranks(start.elapsed_time(end), dev if dist_barrier and _nccl() else None)
    return ms, pipe, stats


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _nccl():
    import torch.distributed as tdist
    return tdist.is_available() and tdist.is_initialized() and tdist.get_backend() == "nccl"


def our_arm(args, world, rank, local):
    import numpy as np
    import torch

    from paper_2112_13169_b200 import _native as N
    from paper_2112_13169_b200 import multi
    from paper_2112_13169_b200 import voxmap as vm
    from tests import scenes

    backend = init_dist(world, local)
    ngpu = torch.cuda.device_count()
    dev_index = local % max(1, ngpu)  # ranks share a GPU when fewer are visible (gloo plumbing)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    barrier = None
    if backend:
        import torch.distributed as tdist
        barrier = tdist.barrier
    c = W.CONFIGS[HEADLINE]
    S = streams_per_rank(args, world)
    K, WU = args.steps, max(3, args.warmup)
    gids = list(multi.stream_range(S, rank))
    npix = c["width"] * c["height"]
    n_cells = W.cells(vm, c)

    wl = Workload(vm, torch, dev, c, gids, pinned=True)
    assert np.array_equal(wl.pool_host[0], scenes.render(W.camera(vm, c), wl.poses[0], _boxes()))

    # ---- device-resident throughput (value): the default batch graphs, whose
    # branches overlap the stages of different stream shares
    clocks = ClockSampler(dev_index)
    ms, pipe, stats = timed_batch(vm, torch, dev, wl, S, K, WU, clocks=clocks, dist_barrier=barrier)
    value = multi.job_throughput(S * K, world, ms / 1000.0)
    branches = pipe.graph_branches
    d = W.dims(vm, c)
    # K1 populate, K2 dilation when vox_inf > 0 (one fused tile kernel when dims_x % 4 == 0, else K2a rows +
    # K2b tiles), K3 trace, K4 merge, per branch; K5 (counter publish) only when K4 is not the direct-load
    # epoch-key merge (rows of more than 1024 cells or not a multiple of 4), which publishes from its last block
    k2 = 0 if c["vox_inf"] == 0 else (1 if d[0] % 4 == 0 else 2)
    k5 = 0 if (d[0] % 4 == 0 and d[0] <= 1024) else 1
    kernels_per_step = (3 + k2 + k5) * branches
    dev_grids, dev_origins = final_state(vm, pipe, S)
    pipe.close()

    # ---- per-kernel device times (the roofline's K3 duration): the same
    # steps as ONE graph branch, stage-boundary events recorded inside the
    # graph on the launching stream, so each stage is timed alone
    kpipe = W.new_pipeline(vm, c, gids, device=dev_index, flags=N.FLAG_SINGLE_BRANCH | N.FLAG_STAGE_EVENTS)
    kstream = torch.cuda.ExternalStream(kpipe.cuda_stream, device=dev)
    for k in range(WU):
        kpipe.integrate_depth_device(*wl.step(k))
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
        kpipe.integrate_depth_device(*wl.step(WU + k))
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
    e2e_pipe = W.new_pipeline(vm, c, gids, device=dev_index)
    for k in range(WU):
        e2e_pipe.integrate_depth_async(*wl.host_step(k))
    e2e_pipe.wait_stats()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    # vxm_integrate_depth_async: pinned host frames -> H2D on the copy stream
    # (double buffered) -> frame graphs -> counters written by K5 into
    # host-mapped memory; the timed region ends when the last frame's stats
    # are on the host.
    t0 = time.perf_counter()
    for k in range(K):
        e2e_pipe.integrate_depth_async(*wl.host_step(WU + k))
    e2e_stats = e2e_pipe.wait_stats()
    e2e_s = time.perf_counter() - t0
    e2e_s = multi.max_over_ranks(e2e_s, dev if _nccl() else None)
    e2e_value = multi.job_throughput(S * K, world, e2e_s)
    h2d = S * npix * 4 + S * 160  # depth frames + per-stream FrameParams
    d2h = S * 96                  # per-stream counters + stage stamps (vxm::kCountersHostBytes)
    e2e_grids, e2e_origins = final_state(vm, e2e_pipe, S)
    e2e_pipe.close()

    # ---- roofline of the dominant kernel (K3): SURVEY §8d algorithmic bytes
    # per frame (4*W*H + 4*N) x the S frames one launch processes / its time
    bytes_per_frame = 4 * npix + 4 * n_cells
    trace_avg_s = statistics.mean(trace_ms) / 1000.0
    achieved = bytes_per_frame * S / trace_avg_s / 1e9
    peak, peak_kind = hbm_peak()
    traffic, prof = profiled_traffic()

    line = {"metric": "frames_per_s", "value": round(value, 1), "unit": "frames/s", "n_gpus": world,
            "steps": K, "warmup": WU, "ms_per_step": round(ms / K, 4), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(c, S, world, args.scaling),
            "e2e": {"value": round(e2e_value, 1), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "stage_ms_per_step": {k: round(v, 4) for k, v in stage_ms.items()},
            "graph_branches": branches,
            "single_branch_ms_per_step": round(single_branch_ms, 4),
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
            "hbm_gbs_pipeline": round(bytes_per_frame * value / world / 1e9, 1)}
    cl = clocks.summary()
    if cl:
        line["clocks"] = cl
    # The step is instruction-issue bound (every kernel but the merge runs at
    # 63-81% issue-active in ncu): its floor is the warp instructions of the
    # five stages over the GPU's issue rate (SMs x 4 schedulers x SM clock).
    si = step_instructions()
    if si and S == 64 and si.get("total"):
        props = torch.cuda.get_device_properties(dev)
        mhz = (cl or {}).get("sm_mhz") or 1965
        floor_ms = si["total"] / (props.multi_processor_count * 4 * mhz * 1e6) * 1e3
        line["issue_roofline"] = {"bound": "warp-instruction issue", "warp_instructions_per_step": int(si["total"]),
                                  "floor_ms_per_step": round(floor_ms, 4), "ms_per_step": round(ms / K, 4),
                                  "frac": round(floor_ms / (ms / K), 4),
                                  "source": si.get("source"), "per_kernel": si.get("warp_instructions")}
    if backend:
        line["dist_backend"] = backend
    wl_pool = wl
    del wl

    # ---- the other configurations and the latency / trajectory numbers
    extras = {}
    if not args.no_extras:
        extras = other_measurements(args, vm, torch, dev, dev_index, world, rank, gids, K, WU, barrier)
        line.update(extras.pop("line", {}))

    # ---- parity of the timed runs and the CPU reference (rank 0)
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import ref_bench
        cores = host_cores()
        if ref_bench.available():
            # the same S streams (this rank's: global ids 0..S-1), WU + K steps
            r = ref_bench.run(c, S, K, WU, cores, pool=W.POOL, y0=W.Y0, dump=True, n_cells=n_cells)
            ok_dev, bad_dev = compare_with_reference(r, dev_grids, dev_origins, stats)
            ok_e2e, bad_e2e = compare_with_reference(r, e2e_grids, e2e_origins, e2e_stats)
            parity = {HEADLINE: {"streams": S, "steps": WU + K, "value_run_match": ok_dev,
                                 "e2e_run_match": ok_e2e, "mismatched_streams": bad_dev + bad_e2e,
                                 "checked": "every stream's final grid bytes and origin, last-step stats"}}
            for name, res in extras.get("parity", {}).items():
                parity[name] = res
            line["parity"] = parity
            line["parity_ok"] = all(v.get("value_run_match", True) and v.get("e2e_run_match", True)
                                    and v.get("match", True) for v in parity.values())
            if world == 1:
                line["cpu_baseline"] = {
                    "value": round(r["frames_per_s"], 3), "unit": "frames/s", "cores": r["threads"],
                    "kind": "reference",
                    "sample": f"{r['frames']} frames ({S} streams x {K} steps after {WU} warm-up, the same pool, "
                              f"rule and start grids), Sequential MappingPipeline per stream, one stream per "
                              f"thread, {cpu_model()}",
                    "latency_ms_p50_under_load": r["p50_ms"]}
                if not args.no_extras:
                    lat = {}
                    for mode, par, thr in (("sequential_1core", False, 1), ("dataparallel_all_cores", True, cores)):
                        q = ref_bench.latency(c, args.latency_frames, par, thr, pool=W.POOL, y0=W.Y0)
                        lat[mode] = {"p50_ms": q["p50_ms"], "p99_ms": q["p99_ms"], "mean_ms": q["mean_ms"],
                                     "frames": q["frames"], "threads": q["threads"]}
                    lat["note"] = ("one stream, depth_to_cloud + MappingPipeline::integrate per frame after 5 "
                                   "warm-up frames (sim::measure); DataParallel = OpenMP rows/rays + AVX2 kernels")
                    line["cpu_baseline"]["latency"] = lat
    if rank == 0:
        print(json.dumps(line), flush=True)
    del wl_pool
    if backend:
        import torch.distributed as tdist
        tdist.barrier()
        tdist.destroy_process_group()


def other_measurements(args, vm, torch, dev, dev_index, world, rank, gids_head, K, WU, barrier):
    """cfg1 x 64 and cfg3 x 16 batches (device-resident, same method as
    `value`), single-stream latency (>= 1000 frames), the cfg4 1000-frame
    sweep, and at N > 1 the strong-scaling split of cfg5's 64 streams."""
    import numpy as np

    from paper_2112_13169_b200 import multi
    from tests import scenes

    out = {"line": {}, "parity": {}}
    configs = {}
    for name, S in (("cfg1", 64), ("cfg3", 16)):
        c = W.CONFIGS[name]
        gids = list(multi.stream_range(S, rank))
        wl = Workload(vm, torch, dev, c, gids)
        ms, pipe, stats = timed_batch(vm, torch, dev, wl, S, K, WU, dist_barrier=barrier)
        grids, origins = final_state(vm, pipe, S)
        pipe.close()
        v = multi.job_throughput(S * K, world, ms / 1000.0)
        d = W.dims(vm, c)
        npix = c["width"] * c["height"]
        configs[name] = {"frames_per_s": round(v, 1), "ms_per_step": round(ms / K, 4), "streams_per_gpu": S,
                         "frame_shape": [c["height"], c["width"]], "grid_dims": list(d),
                         "vox_size": c["vox"], "vox_inf": c["vox_inf"], "depth_m": c["depth"],
                         "hbm_gbs_pipeline": round((4 * npix + 4 * d[0] * d[1] * d[2]) * v / world / 1e9, 1)}
        if rank == 0 and not args.no_cpu_baseline:
            from oracle import ref_bench
            if ref_bench.available():
                r = ref_bench.run(c, S, K, WU, host_cores(), pool=W.POOL, y0=W.Y0, dump=True,
                                  n_cells=d[0] * d[1] * d[2])
                ok, bad = compare_with_reference(r, grids, origins, stats)
                out["parity"][name] = {"streams": S, "steps": WU + K, "match": ok, "mismatched_streams": bad}
                configs[name]["cpu_reference_frames_per_s"] = round(r["frames_per_s"], 1)
        del wl
        torch.cuda.empty_cache()

    # ---- single-stream latency, cfg2, one frame at a time
    c = W.CONFIGS[HEADLINE]
    wl = Workload(vm, torch, dev, c, [0], pinned=True)
    poses = wl.poses
    one_pose = [vm.pose_array([poses[j]]) for j in range(W.POOL)]
    lat = W.new_pipeline(vm, c, [0], device=dev_index)
    dev_lat, e2e_lat = [], []
    n = args.latency_frames
    for k in range(n + 10):
        j = k % W.POOL
        lat.integrate_depth_device(wl.pool_dev[j].data_ptr(), one_pose[j])
        lat.wait_stats()
        if k >= 10:
            dev_lat.append(lat.last_frame_ms())
    lat.close()
    one = torch.empty((1, c["height"], c["width"]), dtype=torch.float32).pin_memory()
    lat = W.new_pipeline(vm, c, [0], device=dev_index)
    for k in range(n + 10):
        j = k % W.POOL
        one[0].copy_(torch.from_numpy(wl.pool_host[j]))
        t1 = time.perf_counter()
        lat.integrate_depth_ptr(one.data_ptr(), one_pose[j])  # synchronous: H2D, graph, stats on the host
        if k >= 10:
            e2e_lat.append((time.perf_counter() - t1) * 1000.0)
    lat.close()
    out["line"]["latency_ms"] = {"p50": round(pct(dev_lat, 0.5), 4), "p99": round(pct(dev_lat, 0.99), 4),
                                 "e2e_p50": round(pct(e2e_lat, 0.5), 4), "e2e_p99": round(pct(e2e_lat, 0.99), 4),
                                 "frames": len(dev_lat),
                                 "note": "cfg2, one stream, one frame at a time; device = CUDA events around the "
                                         "frame's graph, e2e = wall time of vxm_integrate_depth from a pinned "
                                         "host frame until the stats are on the host"}
    del wl

    # ---- cfg4: sim::sweep_trajectory((0,-50,0),(0,50,0),1000) on cfg1 frames
    # through the corridor scene, device-resident frames rendered on the GPU
    c1 = W.CONFIGS["cfg1"]
    cam = W.camera(vm, c1)
    positions = W.sweep_positions(1000)
    traj_poses = [vm.look_along_x(p) for p in positions]
    frames = torch.empty((1000, c1["height"], c1["width"]), dtype=torch.float32, device=dev)
    vm.render_depth(cam, traj_poses, scenes.corridor_boxes(-60.0, 60.0), out_ptr=frames.data_ptr(), device=dev_index)
    torch.cuda.synchronize()
    cfg4 = vm.PipelineConfig(W.grid_for(vm, c1, positions[0]), cam, vox_inf=c1["vox_inf"], depth=c1["depth"])
    F = 64
    full_calls = 1000 // F
    pa = [vm.pose_array(traj_poses[i * F:(i + 1) * F]) for i in range(full_calls)]
    tail = 1000 - full_calls * F
    seq = vm.MappingPipeline(cfg4, frames_per_call=F, device=dev_index)
    single = vm.MappingPipeline(cfg4, device=dev_index)
    one_pa = [vm.pose_array([p]) for p in traj_poses]
    tail_host = frames[full_calls * F:].cpu().numpy()
    res = {}
    for rep in range(2):
        # the first pass warms the pipelines up (graph capture, lazy module
        # loading), the second is timed on the same pipelines: it starts with
        # a 100 m jump back to the trajectory's start (a full grid reset) and
        # then does the first pass's work frame for frame
        st = torch.cuda.ExternalStream(seq.cuda_stream, device=dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record(st)
        for i in range(full_calls):
            seq.integrate_depth_device(frames[i * F].data_ptr(), pa[i])
        b.record(st)
        seq.wait_stats()
        seq_dev_ms = a.elapsed_time(b)
        seq.integrate_depth_frames(tail_host, traj_poses[full_calls * F:])  # the last 40 frames (host call)
        seq_wall = time.perf_counter() - t0
        st1 = torch.cuda.ExternalStream(single.cuda_stream, device=dev)
        a1, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a1.record(st1)
        for i in range(1000):
            single.integrate_depth_device(frames[i].data_ptr(), one_pa[i])
        b1.record(st1)
        last = single.wait_stats()
        single_ms = a1.elapsed_time(b1)
        res = {"frames": 1000, "multi_frame_frames_per_s": round(full_calls * F / (seq_dev_ms / 1000.0), 1),
               "multi_frame_wall_s_all_1000": round(seq_wall, 4),
               "single_frame_frames_per_s": round(1000 / (single_ms / 1000.0), 1),
               "single_frame_us_per_frame": round(single_ms * 1000.0 / 1000, 3),
               "final_origin": [round(x, 6) for x in last[0]["origin"]],
               "grids_equal_multi_vs_single": bool(np.array_equal(seq.local_grid()[0], single.local_grid()[0])),
               "note": "one robot; multi_frame = 15 calls of 64 consecutive frames (chain-folded merge, device "
                       "frames, CUDA events) + the last 40 frames as a host call in the wall time; single_frame = "
                       "1000 back-to-back one-frame calls on device frames; each the second of two passes over the "
                       "trajectory on the same pipeline (the first warms it up); full-size parity vs the "
                       "reference: tests/test_gpu_trajectory.py"}
    seq.close()
    single.close()
    del frames
    torch.cuda.empty_cache()
    configs["cfg4"] = res

    # ---- strong scaling of cfg5 as written (64 streams in total, 64/N per GPU)
    if world > 1 and 64 % world == 0:
        c = W.CONFIGS[HEADLINE]
        Sg = 64 // world
        gids = list(multi.stream_range(Sg, rank))
        wl = Workload(vm, torch, dev, c, gids)
        ms, pipe, _ = timed_batch(vm, torch, dev, wl, Sg, K, WU, dist_barrier=barrier)
        pipe.close()
        configs["cfg5_strong"] = {"streams_total": 64, "streams_per_gpu": Sg,
                                  "frames_per_s": round(multi.job_throughput(Sg * K, world, ms / 1000.0), 1),
                                  "ms_per_step": round(ms / K, 4)}
        del wl
    out["line"]["configs"] = configs
    return out


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    from paper_2112_13169_b200 import multi
    world, rank, local = multi.env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.plumbing_only:
        plumbing_arm(args, world, rank, local)
    elif args.impl == "reference":
        reference_arm(args, world, rank)
    else:
        our_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
