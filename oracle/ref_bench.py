"""ORACLE / TEST INFRASTRUCTURE ONLY.

Runs oracle/_ref/ref_bench (the UNMODIFIED reference sources, oracle/ref_bench.cpp
driver) on the benchmark workload of tests/workload.py and reads back its
parity dumps. Used by tests/ (parity of the exact benchmarked workload) and by
bench.py's cpu_baseline leg / reference arm (the timed CPU reference, and the
checker of the GPU run's final grids). The product never imports it.
"""
from __future__ import annotations

import json
import os
import subprocess
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
EXE = ROOT / "_ref" / "ref_bench"
STAT_KEYS = ("points_total", "points_outside", "rays_traced", "voxels_freed", "voxels_marked_unknown_traced",
             "voxels_skipped_out_of_bounds", "occupied_count", "freed_count", "shifted")


def available() -> bool:
    return EXE.exists()


def _cfg_args(c, pool, y0):
    return ["--width", str(c["width"]), "--height", str(c["height"]), "--vox", repr(c["vox"]),
            "--gx", repr(c["grid"][0]), "--gy", repr(c["grid"][1]), "--gz", repr(c["grid"][2]),
            "--depth", repr(c["depth"]), "--vox-inf", str(c["vox_inf"]), "--pool", str(pool), "--y0", repr(y0)]


def run(c, streams, steps, warmup, threads, pool=16, y0=-0.8, dump=False, n_cells=None, timeout=1800):
    """Throughput run: `streams` Sequential pipelines over `threads` host
    threads, `warmup` untimed + `steps` timed steps. With dump=True also
    returns every step's per-stream stats (warm-up included) as an int64
    array (warmup + steps, streams, 9) in STAT_KEYS order, the final grids
    (streams, n_cells) and their origins (streams, 3)."""
    if not available():
        return None
    cmd = [str(EXE), *_cfg_args(c, pool, y0), "--streams", str(streams), "--steps", str(steps),
           "--warmup", str(warmup), "--threads", str(threads)]
    with tempfile.TemporaryDirectory() as td:
        st_path, gr_path = os.path.join(td, "stats.bin"), os.path.join(td, "grids.bin")
        if dump:
            cmd += ["--dump-stats", st_path, "--dump-grids", gr_path]
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        if out.returncode != 0:
            raise RuntimeError(f"ref_bench failed ({out.returncode}): {out.stderr[-500:]}")
        res = json.loads(out.stdout.strip().splitlines()[-1])
        if dump:
            res["stats"] = np.fromfile(st_path, dtype=np.int64).reshape(warmup + steps, streams, 9)
            raw = np.fromfile(gr_path, dtype=np.uint8)
            n = (raw.size - 24 * streams) // streams if n_cells is None else n_cells
            res["grids"] = raw[: n * streams].reshape(streams, n)
            res["origins"] = raw[n * streams:].view(np.float64).reshape(streams, 3)
    return res


def latency(c, frames, parallel, threads, pool=16, y0=-0.8, timeout=1800):
    """One stream, `frames` frames after 5 warm-up frames (sim::measure):
    Sequential on one core, or DataParallel over `threads` OpenMP threads."""
    if not available():
        return None
    cmd = [str(EXE), *_cfg_args(c, pool, y0), "--latency-frames", str(frames), "--parallel",
           "1" if parallel else "0", "--threads", str(threads)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    if out.returncode != 0:
        raise RuntimeError(f"ref_bench failed ({out.returncode}): {out.stderr[-500:]}")
    return json.loads(out.stdout.strip().splitlines()[-1])


def stats_row(d) -> list:
    """a voxmap stats dict in STAT_KEYS order"""
    return [int(d[k]) for k in STAT_KEYS]
