"""ctypes binding of the C-ABI in include/vxm.h (libvxm.so, built in-tree).

This is the Python face of the drop-in boundary: the same entry points a
cgo / JNI / ctypes caller of the reference path would bind.
There is no CPU fallback: if libvxm.so is missing or no sm_100 GPU is
visible, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "lib" / os.environ.get("VXM_LIB_NAME", "libvxm.so")  # override: A/B builds

VXM_OK, VXM_EINVAL, VXM_ECUDA, VXM_ENOMEM, VXM_ENODEV, VXM_ESTATE, VXM_EIO = range(7)
UNKNOWN, FREE, OCCUPIED, UNKNOWN_TRACED = 0, 1, 2, 3
TRACER_BUNDLED, TRACER_PER_PIXEL = 0, 1
FLAG_STAGE_TIMING, FLAG_NO_GRAPH, FLAG_SINGLE_BRANCH, FLAG_NO_TMA_MERGE, FLAG_STAGE_EVENTS = 1, 2, 4, 8, 16
FLAG_NO_DESYNC = 32
FLAG_CLEAR_KEYS = 64


class GridSpecC(C.Structure):
    _fields_ = [("size", C.c_double * 3), ("vox_size", C.c_double), ("dims", C.c_int32 * 3),
                ("pad_", C.c_int32), ("origin", C.c_double * 3)]


class CameraC(C.Structure):
    _fields_ = [("fov_x", C.c_double), ("fov_y", C.c_double), ("width", C.c_int32),
                ("height", C.c_int32), ("max_depth", C.c_double)]


class ConfigC(C.Structure):
    _fields_ = [("grid", GridSpecC), ("camera", CameraC), ("vox_inf", C.c_int32),
                ("tracer_mode", C.c_int32), ("depth", C.c_double)]


class PoseC(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("translation", C.c_double * 3)]


class StatsC(C.Structure):
    _fields_ = [("points_total", C.c_uint64), ("points_outside", C.c_uint64),
                ("rays_traced", C.c_uint64), ("voxels_freed", C.c_uint64),
                ("voxels_marked_unknown_traced", C.c_uint64),
                ("voxels_skipped_out_of_bounds", C.c_uint64), ("occupied_count", C.c_uint64),
                ("freed_count", C.c_uint64), ("shifted", C.c_int32),
                ("shift_offset", C.c_int32 * 3), ("origin", C.c_double * 3),
                ("populate_us", C.c_double), ("trace_us", C.c_double), ("merge_us", C.c_double),
                ("shift_us", C.c_double)]


class PopulateStatsC(C.Structure):
    _fields_ = [("points_total", C.c_uint64), ("points_outside", C.c_uint64)]


class TraceStatsC(C.Structure):
    _fields_ = [("rays_traced", C.c_uint64), ("voxels_freed", C.c_uint64),
                ("voxels_marked_unknown_traced", C.c_uint64),
                ("voxels_skipped_out_of_bounds", C.c_uint64)]


P = C.POINTER
_u8p, _f32p, _f64p, _i32p = P(C.c_uint8), P(C.c_float), P(C.c_double), P(C.c_int32)

# name -> (restype, argtypes); every symbol include/vxm.h declares.
SIGNATURES = {
    "vxm_grid_spec_create": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, _f64p, P(GridSpecC)]),
    "vxm_grid_spec_create_centered": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, _f64p, P(GridSpecC)]),
    "vxm_bundle_dimensions": (C.c_int, [P(CameraC), C.c_double, C.c_double, _i32p]),
    "vxm_last_error": (C.c_char_p, []),
    "vxm_build_info": (C.c_char_p, []),
    "vxm_device_count": (C.c_int, []),
    "vxm_create": (C.c_int, [P(ConfigC), C.c_int32, C.c_int32, C.c_uint32, P(C.c_void_p)]),
    "vxm_destroy": (C.c_int, [C.c_void_p]),
    "vxm_num_streams": (C.c_int, [C.c_void_p]),
    "vxm_create_multi": (C.c_int, [P(ConfigC), C.c_int32, C.c_int32, C.c_int32, C.c_uint32, P(C.c_void_p)]),
    "vxm_frames_per_call": (C.c_int, [C.c_void_p]),
    "vxm_graph_branches": (C.c_int, [C.c_void_p]),
    "vxm_grid_write": (C.c_int, [C.c_char_p, P(GridSpecC), C.c_void_p]),
    "vxm_render_depth": (C.c_int, [P(CameraC), P(PoseC), C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]),
    "vxm_grid_read": (C.c_int, [C.c_char_p, P(GridSpecC), C.c_void_p, C.c_size_t]),
    "vxm_snapshot_save": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p]),
    "vxm_snapshot_load": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p]),
    "vxm_snapshot_save_async": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p]),
    "vxm_snapshot_wait": (C.c_int, [C.c_void_p]),
    "vxm_integrate_depth_frames": (C.c_int, [C.c_void_p, C.c_void_p, P(PoseC), C.c_int32, P(StatsC)]),
    "vxm_integrate_depth": (C.c_int, [C.c_void_p, C.c_void_p, P(PoseC), P(StatsC)]),
    "vxm_integrate_depth_device": (C.c_int, [C.c_void_p, C.c_void_p, P(PoseC)]),
    "vxm_wait_stats": (C.c_int, [C.c_void_p, P(StatsC)]),
    "vxm_integrate_depth_async": (C.c_int, [C.c_void_p, C.c_void_p, P(PoseC)]),
    "vxm_integrate_cloud": (C.c_int, [C.c_void_p, _f64p, _f64p, _f64p, C.c_size_t, P(PoseC), P(StatsC)]),
    "vxm_download_local": (C.c_int, [C.c_void_p, C.c_int32, _u8p, _f64p]),
    "vxm_upload_local": (C.c_int, [C.c_void_p, C.c_int32, _u8p, _f64p]),
    "vxm_cuda_stream": (C.c_void_p, [C.c_void_p]),
    "vxm_last_frame_ms": (C.c_int, [C.c_void_p, P(C.c_float)]),
    "vxm_set_input_event": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vxm_set_stage_events": (C.c_int, [C.c_void_p, P(C.c_void_p)]),
    "vxm_populate_occupied": (C.c_int, [P(GridSpecC), _u8p, _f64p, _f64p, _f64p, C.c_size_t, P(PoseC), C.c_int32, P(PopulateStatsC)]),
    "vxm_trace_bundle": (C.c_int, [P(GridSpecC), _u8p, _i32p, P(PoseC), C.c_double, P(TraceStatsC)]),
    "vxm_trace_per_pixel": (C.c_int, [P(GridSpecC), _u8p, _f64p, _f64p, _f64p, C.c_size_t, P(PoseC), P(TraceStatsC)]),
    "vxm_merge_grids": (C.c_int, [_u8p, _u8p, C.c_size_t]),
    "vxm_shift_grid": (C.c_int, [_i32p, _u8p, _u8p, _i32p]),
    "vxm_depth_to_cloud": (C.c_int, [P(CameraC), _f32p, _f64p, _f64p, _f64p, P(C.c_size_t)]),
    "vxm_kernel_merge": (None, [_u8p, _u8p, C.c_size_t]),
    "vxm_kernel_transform_voxelize": (None, [_f64p, _f64p, _f64p, C.c_size_t, _f64p, _f64p, C.c_double, _i32p, _i32p, _i32p]),
    "vxm_kernel_isa": (C.c_char_p, []),
}

_lib = None


def load() -> C.CDLL:
    """Load libvxm.so (in-tree build). Raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(os.fspath(LIB_PATH))
        lenient = os.environ.get("VXM_LIB_NAME") is not None  # A/B builds of older revisions
        for name, (res, args) in SIGNATURES.items():
            if lenient and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class VxmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"vxm error {code}: {msg}")
        self.code = code


def check(rc: int) -> None:
    """Map a vxm status to the reference's exception types."""
    if rc == VXM_OK:
        return
    msg = (load().vxm_last_error() or b"").decode()
    if rc == VXM_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    raise VxmError(rc, msg)
