"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_ref/libvoxmap_ref.so: the UNMODIFIED reference
voxmap sources (proj/src) compiled against the in-repo Eigen subset by
oracle/Makefile.ref, plus the flat C shim oracle/ref_capi.cpp. Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may use
this module; the product never imports it.

All grids are numpy uint8 arrays in the reference cell order; poses are
(R 3x3, t 3) pairs; structs are the vxm.h PODs from paper_2112_13169_b200._native.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from paper_2112_13169_b200 import _native as N

ROOT = Path(__file__).resolve().parent
LIB_PATH = ROOT / "_ref" / "libvoxmap_ref.so"

P = C.POINTER
_u8p, _f32p, _f64p, _i32p = P(C.c_uint8), P(C.c_float), P(C.c_double), P(C.c_int32)

SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_dispatch_isa": (C.c_char_p, []),
    "ref_grid_spec_create_centered": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, _f64p, P(N.GridSpecC)]),
    "ref_bundle_dimensions": (C.c_int, [P(N.CameraC), C.c_double, C.c_double, _i32p]),
    "ref_look_along_x": (C.c_int, [_f64p, P(N.PoseC)]),
    "ref_render_depth": (C.c_int, [C.c_int, C.c_uint64, _f64p, C.c_int, P(N.PoseC), P(N.CameraC), C.c_int, _f32p]),
    "ref_box_field": (C.c_int, [C.c_uint64, _f64p, P(C.c_int)]),
    "ref_depth_to_cloud": (C.c_int, [P(N.CameraC), _f32p, C.c_int, _f64p, _f64p, _f64p, P(C.c_size_t)]),
    "ref_merge": (None, [_u8p, _u8p, C.c_size_t, C.c_int]),
    "ref_transform_voxelize": (None, [_f64p, _f64p, _f64p, C.c_size_t, _f64p, _f64p, C.c_double, _i32p, _i32p, _i32p, C.c_int]),
    "ref_populate": (C.c_int, [P(N.GridSpecC), _u8p, _f64p, _f64p, _f64p, C.c_size_t, P(N.PoseC), C.c_int, C.c_int, P(N.PopulateStatsC)]),
    "ref_trace_bundle": (C.c_int, [P(N.GridSpecC), _u8p, _i32p, P(N.PoseC), C.c_int, P(N.TraceStatsC)]),
    "ref_trace_per_pixel": (C.c_int, [P(N.GridSpecC), _u8p, _f64p, _f64p, _f64p, C.c_size_t, P(N.PoseC), P(N.TraceStatsC)]),
    "ref_shift": (C.c_int, [P(N.GridSpecC), _u8p, _u8p, _i32p]),
    "ref_write_grid": (C.c_int, [P(N.GridSpecC), _u8p, C.c_char_p]),
    "ref_read_grid": (C.c_int, [C.c_char_p, P(N.GridSpecC), C.c_void_p, C.c_size_t]),
    "ref_pipeline_create": (C.c_void_p, [P(N.ConfigC), C.c_int]),
    "ref_pipeline_destroy": (None, [C.c_void_p]),
    "ref_pipeline_integrate_cloud": (C.c_int, [C.c_void_p, _f64p, _f64p, _f64p, C.c_size_t, P(N.PoseC), P(N.StatsC)]),
    "ref_pipeline_integrate_depth": (C.c_int, [C.c_void_p, _f32p, P(N.PoseC), P(N.StatsC)]),
    "ref_pipeline_local": (C.c_int, [C.c_void_p, _u8p, _f64p]),
}

_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} not built (make -f oracle/Makefile.ref)")
        L = C.CDLL(os.fspath(LIB_PATH))
        for k, (r, a) in SIGS.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise ValueError(lib().ref_last_error().decode())


def _f64(a):
    return a.ctypes.data_as(_f64p)


def _u8(a):
    return a.ctypes.data_as(_u8p)


def _i32(a):
    return a.ctypes.data_as(_i32p)


def _f32(a):
    return a.ctypes.data_as(_f32p)


def pose_c(pose):
    from paper_2112_13169_b200.voxmap import pose_c as pc
    return pc(pose)


def render_depth(cam_c, pose, scene="boxes", seed=1, boxes=None, parallel=True):
    out = np.empty(cam_c.height * cam_c.width, dtype=np.float32)
    kind = {"empty": 0, "wall": 1, "boxes": 2}[scene] if boxes is None else 0
    bx = None if boxes is None else np.ascontiguousarray(boxes, dtype=np.float64)
    _check(lib().ref_render_depth(kind, seed, None if bx is None else _f64(bx), 0 if bx is None else len(bx),
                                  C.byref(pose_c(pose)), C.byref(cam_c), 1 if parallel else 0, _f32(out)))
    return out.reshape(cam_c.height, cam_c.width)


def box_field(seed):
    out = np.empty((16, 6), dtype=np.float64)
    n = C.c_int()
    _check(lib().ref_box_field(seed, _f64(out), C.byref(n)))
    return out[: n.value].copy()


def depth_to_cloud(cam_c, depth, parallel=False):
    depth = np.ascontiguousarray(depth, dtype=np.float32)
    n = depth.size
    xs, ys, zs = (np.empty(n) for _ in range(3))
    cnt = C.c_size_t()
    _check(lib().ref_depth_to_cloud(C.byref(cam_c), _f32(depth), 1 if parallel else 0, _f64(xs), _f64(ys),
                                    _f64(zs), C.byref(cnt)))
    k = cnt.value
    return xs[:k].copy(), ys[:k].copy(), zs[:k].copy()


def merge(local, ms, use_dispatch=False):
    lib().ref_merge(_u8(local), _u8(ms), local.size, 1 if use_dispatch else 0)


def transform_voxelize(xs, ys, zs, R, t, vs, use_dispatch=False):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    R = np.ascontiguousarray(R, dtype=np.float64).reshape(9)
    t = np.ascontiguousarray(t, dtype=np.float64).reshape(3)
    n = len(xs)
    cx, cy, cz = (np.empty(n, dtype=np.int32) for _ in range(3))
    lib().ref_transform_voxelize(_f64(xs), _f64(ys), _f64(zs), n, _f64(R), _f64(t), vs, _i32(cx), _i32(cy),
                                 _i32(cz), 1 if use_dispatch else 0)
    return cx, cy, cz


def populate(grid_c, ms, xs, ys, zs, t_vc, vox_inf, parallel=False):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    st = N.PopulateStatsC()
    _check(lib().ref_populate(C.byref(grid_c), _u8(ms), _f64(xs), _f64(ys), _f64(zs), len(xs),
                              C.byref(pose_c(t_vc)), vox_inf, 1 if parallel else 0, C.byref(st)))
    return {"points_total": st.points_total, "points_outside": st.points_outside}


def trace_bundle(grid_c, ms, bundle, t_vc, parallel=False):
    b = np.asarray(bundle, dtype=np.int32)
    st = N.TraceStatsC()
    _check(lib().ref_trace_bundle(C.byref(grid_c), _u8(ms), _i32(b), C.byref(pose_c(t_vc)), 1 if parallel else 0,
                                  C.byref(st)))
    return {k: getattr(st, k) for k, _ in N.TraceStatsC._fields_}


def trace_per_pixel(grid_c, ms, xs, ys, zs, t_vc):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    st = N.TraceStatsC()
    _check(lib().ref_trace_per_pixel(C.byref(grid_c), _u8(ms), _f64(xs), _f64(ys), _f64(zs), len(xs),
                                     C.byref(pose_c(t_vc)), C.byref(st)))
    return {k: getattr(st, k) for k, _ in N.TraceStatsC._fields_}


def shift(grid_c, cells, off):
    out = np.empty_like(cells)
    o = np.asarray(off, dtype=np.int32)
    _check(lib().ref_shift(C.byref(grid_c), _u8(cells), _u8(out), _i32(o)))
    return out


def write_grid(grid_c, cells, path):
    cells = np.ascontiguousarray(cells, dtype=np.uint8)
    _check(lib().ref_write_grid(C.byref(grid_c), _u8(cells), str(path).encode()))


def read_grid(path):
    """-> (GridSpecC, cells) through the reference's read_grid"""
    g = N.GridSpecC()
    _check(lib().ref_read_grid(str(path).encode(), C.byref(g), None, 0))
    cells = np.empty(g.dims[0] * g.dims[1] * g.dims[2], dtype=np.uint8)
    _check(lib().ref_read_grid(str(path).encode(), C.byref(g), cells.ctypes.data, cells.size))
    return g, cells


class Pipeline:
    """MappingPipeline from the reference library (Sequential by default: the
    bit-exact parity mode)."""

    def __init__(self, cfg_c, parallel=False):
        self._p = lib().ref_pipeline_create(C.byref(cfg_c), 1 if parallel else 0)
        if not self._p:
            raise ValueError(lib().ref_last_error().decode())
        self.n = cfg_c.grid.dims[0] * cfg_c.grid.dims[1] * cfg_c.grid.dims[2]
        self._st = N.StatsC()

    def __del__(self):
        if getattr(self, "_p", None):
            lib().ref_pipeline_destroy(self._p)
            self._p = None

    def integrate_depth(self, depth, pose):
        depth = np.ascontiguousarray(depth, dtype=np.float32)
        _check(lib().ref_pipeline_integrate_depth(self._p, _f32(depth), C.byref(pose_c(pose)), C.byref(self._st)))
        from paper_2112_13169_b200.voxmap import stats_dict
        return stats_dict(self._st)

    def integrate(self, xs, ys, zs, pose):
        xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
        _check(lib().ref_pipeline_integrate_cloud(self._p, _f64(xs), _f64(ys), _f64(zs), len(xs),
                                                  C.byref(pose_c(pose)), C.byref(self._st)))
        from paper_2112_13169_b200.voxmap import stats_dict
        return stats_dict(self._st)

    def local_grid(self):
        cells = np.empty(self.n, dtype=np.uint8)
        origin = np.empty(3)
        _check(lib().ref_pipeline_local(self._p, _u8(cells), _f64(origin)))
        return cells, origin
