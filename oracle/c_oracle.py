"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper of the plain-C restatement oracle/voxmap_oracle.c
(oracle/build/liboracle.so, built by paper_2112_13169_b200.build.build_oracle
or on demand here with gcc). Same call shapes as oracle/ref.py so tests can
check against either.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2112_13169_b200 import _native as N

ROOT = Path(__file__).resolve().parent
SRC = ROOT / "voxmap_oracle.c"
LIB_PATH = ROOT / "build" / "liboracle.so"

P = C.POINTER
_u8p, _f32p, _f64p, _i32p = P(C.c_uint8), P(C.c_float), P(C.c_double), P(C.c_int32)
SIGS = {
    "vo_merge": (None, [_u8p, _u8p, C.c_size_t]),
    "vo_transform_voxelize": (None, [_f64p, _f64p, _f64p, C.c_size_t, _f64p, _f64p, C.c_double, _i32p, _i32p, _i32p]),
    "vo_depth_to_cloud": (C.c_longlong, [P(N.CameraC), _f32p, _f64p, _f64p, _f64p]),
    "vo_populate": (C.c_int, [P(N.GridSpecC), _u8p, _f64p, _f64p, _f64p, C.c_size_t, P(N.PoseC), C.c_int, P(N.PopulateStatsC)]),
    "vo_bundle_dimensions": (C.c_int, [P(N.CameraC), C.c_double, C.c_double, _i32p]),
    "vo_trace_bundle": (C.c_int, [P(N.GridSpecC), _u8p, _i32p, P(N.PoseC), P(N.TraceStatsC)]),
    "vo_trace_per_pixel": (C.c_int, [P(N.GridSpecC), _u8p, _f64p, _f64p, _f64p, C.c_size_t, P(N.PoseC), P(N.TraceStatsC)]),
    "vo_shift": (None, [_i32p, _u8p, _u8p, _i32p]),
    "vo_pipeline_create": (C.c_void_p, [P(N.ConfigC)]),
    "vo_pipeline_destroy": (None, [C.c_void_p]),
    "vo_pipeline_integrate_cloud": (C.c_int, [C.c_void_p, _f64p, _f64p, _f64p, C.c_size_t, P(N.PoseC), P(N.StatsC)]),
    "vo_pipeline_integrate_depth": (C.c_int, [C.c_void_p, _f32p, P(N.PoseC), P(N.StatsC)]),
    "vo_pipeline_local": (None, [C.c_void_p, _u8p, _f64p]),
}
_lib = None


def build():
    LIB_PATH.parent.mkdir(exist_ok=True)
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-Wall",
                        str(SRC), "-o", str(LIB_PATH), "-lm"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(os.fspath(LIB_PATH))
        for k, (r, a) in SIGS.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _f64(a):
    return a.ctypes.data_as(_f64p)


def _u8(a):
    return a.ctypes.data_as(_u8p)


def _i32(a):
    return a.ctypes.data_as(_i32p)


def _pose(p):
    from paper_2112_13169_b200.voxmap import pose_c
    return pose_c(p)


def merge(local, ms):
    lib().vo_merge(_u8(local), _u8(ms), local.size)


def transform_voxelize(xs, ys, zs, R, t, vs):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    R = np.ascontiguousarray(R, dtype=np.float64).reshape(9)
    t = np.ascontiguousarray(t, dtype=np.float64).reshape(3)
    n = len(xs)
    out = [np.empty(n, dtype=np.int32) for _ in range(3)]
    lib().vo_transform_voxelize(_f64(xs), _f64(ys), _f64(zs), n, _f64(R), _f64(t), vs, *(_i32(o) for o in out))
    return tuple(out)


def depth_to_cloud(cam_c, depth):
    depth = np.ascontiguousarray(depth, dtype=np.float32)
    xs, ys, zs = (np.empty(depth.size) for _ in range(3))
    n = lib().vo_depth_to_cloud(C.byref(cam_c), depth.ctypes.data_as(_f32p), _f64(xs), _f64(ys), _f64(zs))
    if n < 0:
        raise ValueError("invalid camera")
    return xs[:n].copy(), ys[:n].copy(), zs[:n].copy()


def populate(grid_c, ms, xs, ys, zs, t_vc, vox_inf):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    st = N.PopulateStatsC()
    if lib().vo_populate(C.byref(grid_c), _u8(ms), _f64(xs), _f64(ys), _f64(zs), len(xs), C.byref(_pose(t_vc)),
                         vox_inf, C.byref(st)):
        raise ValueError("populate precondition")
    return {"points_total": st.points_total, "points_outside": st.points_outside}


def bundle_dimensions(cam_c, depth, vs):
    out = (C.c_int32 * 3)()
    if lib().vo_bundle_dimensions(C.byref(cam_c), depth, vs, out):
        raise ValueError("bundle precondition")
    return tuple(out)


def trace_bundle(grid_c, ms, bundle, t_vc):
    b = np.asarray(bundle, dtype=np.int32)
    st = N.TraceStatsC()
    if lib().vo_trace_bundle(C.byref(grid_c), _u8(ms), _i32(b), C.byref(_pose(t_vc)), C.byref(st)):
        raise ValueError("trace precondition")
    return {k: getattr(st, k) for k, _ in N.TraceStatsC._fields_}


def trace_per_pixel(grid_c, ms, xs, ys, zs, t_vc):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    st = N.TraceStatsC()
    if lib().vo_trace_per_pixel(C.byref(grid_c), _u8(ms), _f64(xs), _f64(ys), _f64(zs), len(xs),
                                C.byref(_pose(t_vc)), C.byref(st)):
        raise ValueError("trace precondition")
    return {k: getattr(st, k) for k, _ in N.TraceStatsC._fields_}


def shift(grid_c, cells, off):
    out = np.empty_like(cells)
    d = np.asarray(grid_c.dims[:], dtype=np.int32)
    o = np.asarray(off, dtype=np.int32)
    lib().vo_shift(_i32(d), _u8(cells), _u8(out), _i32(o))
    return out


class Pipeline:
    """Sequential MappingPipeline restatement."""

    def __init__(self, cfg_c):
        self._p = lib().vo_pipeline_create(C.byref(cfg_c))
        if not self._p:
            raise ValueError("invalid PipelineConfig")
        self.n = cfg_c.grid.dims[0] * cfg_c.grid.dims[1] * cfg_c.grid.dims[2]
        self._st = N.StatsC()

    def __del__(self):
        if getattr(self, "_p", None):
            lib().vo_pipeline_destroy(self._p)
            self._p = None

    def integrate_depth(self, depth, pose):
        from paper_2112_13169_b200.voxmap import stats_dict
        depth = np.ascontiguousarray(depth, dtype=np.float32)
        if lib().vo_pipeline_integrate_depth(self._p, depth.ctypes.data_as(_f32p), C.byref(_pose(pose)),
                                             C.byref(self._st)):
            raise ValueError("MeasurementFrame: invalid transform")
        return stats_dict(self._st)

    def integrate(self, xs, ys, zs, pose):
        from paper_2112_13169_b200.voxmap import stats_dict
        xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
        if lib().vo_pipeline_integrate_cloud(self._p, _f64(xs), _f64(ys), _f64(zs), len(xs), C.byref(_pose(pose)),
                                             C.byref(self._st)):
            raise ValueError("MeasurementFrame: invalid transform")
        return stats_dict(self._st)

    def local_grid(self):
        cells = np.empty(self.n, dtype=np.uint8)
        origin = np.empty(3)
        lib().vo_pipeline_local(self._p, _u8(cells), _f64(origin))
        return cells, origin
