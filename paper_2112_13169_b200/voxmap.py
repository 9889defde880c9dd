"""Python mirror of the reference voxmap API for the per-frame path
(proj/include/voxmap/{grid,geometry,integrator,raytracer,pipeline}.hpp),
driving the sm_100a kernels through the C-ABI (include/vxm.h).

Names, argument meaning and error behaviour follow the reference:
precondition violations raise ValueError (std::invalid_argument). Grids are
numpy uint8 arrays in the reference's flat cell order
idx = x + y*dims_x + z*dims_x*dims_y (grid.hpp:72-77). Poses are
(R 3x3, t 3) pairs, p' = R p + t.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

UNKNOWN, FREE, OCCUPIED, UNKNOWN_TRACED = N.UNKNOWN, N.FREE, N.OCCUPIED, N.UNKNOWN_TRACED


def _f64(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _i32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def pose_c(pose) -> N.PoseC:
    R, t = pose
    R = np.asarray(R, dtype=np.float64).reshape(3, 3)
    t = np.asarray(t, dtype=np.float64).reshape(3)
    p = N.PoseC()
    for i in range(9):
        p.rotation[i] = float(R.flat[i])
    for i in range(3):
        p.translation[i] = float(t[i])
    return p


def pose_array(poses) -> np.ndarray:
    """Poses as one (n, 12) float64 array in vxm_pose layout (rotation
    row-major, then translation): the form the batched calls take without
    per-pose marshalling."""
    out = np.empty((len(poses), 12), dtype=np.float64)
    for i, (R, t) in enumerate(poses):
        out[i, :9] = np.asarray(R, dtype=np.float64).reshape(9)
        out[i, 9:] = np.asarray(t, dtype=np.float64).reshape(3)
    return out


def look_along_x(position):
    """sim::look_along_x (proj/src/sim/trajectory.cpp:7-13): optical axis +x,
    image right -y, image down -z."""
    R = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
    return R, np.asarray(position, dtype=np.float64)


def identity_pose(t=(0.0, 0.0, 0.0)):
    return np.eye(3), np.asarray(t, dtype=np.float64)


@dataclass
class CameraModel:
    """CameraModel (geometry.hpp:60-72); fov in radians."""
    fov_x: float = 85.0 * math.pi / 180.0
    fov_y: float = 101.0 * math.pi / 180.0
    width: int = 320
    height: int = 240
    max_depth: float = 6.5

    def to_c(self) -> N.CameraC:
        return N.CameraC(self.fov_x, self.fov_y, self.width, self.height, self.max_depth)

    def focal_x(self):
        return (self.width / 2.0) / math.tan(self.fov_x / 2.0)

    def focal_y(self):
        return (self.height / 2.0) / math.tan(self.fov_y / 2.0)


class GridSpec:
    """GridSpec (grid.hpp:27-68) backed by the C struct."""

    def __init__(self, c: N.GridSpecC):
        self.c = c

    @staticmethod
    def create(sx, sy, sz, vox_size, origin=(0.0, 0.0, 0.0)) -> "GridSpec":
        c = N.GridSpecC()
        o = np.asarray(origin, dtype=np.float64)
        N.check(N.load().vxm_grid_spec_create(sx, sy, sz, vox_size, _f64(o), C.byref(c)))
        return GridSpec(c)

    @staticmethod
    def create_centered(sx, sy, sz, vox_size, center) -> "GridSpec":
        c = N.GridSpecC()
        o = np.asarray(center, dtype=np.float64)
        N.check(N.load().vxm_grid_spec_create_centered(sx, sy, sz, vox_size, _f64(o), C.byref(c)))
        return GridSpec(c)

    @property
    def dims(self):
        return tuple(self.c.dims)

    @property
    def vox_size(self):
        return self.c.vox_size

    @property
    def origin(self):
        return np.array(self.c.origin[:])

    def cell_count(self):
        d = self.dims
        return d[0] * d[1] * d[2]


@dataclass
class PipelineConfig:
    """PipelineConfig (pipeline.hpp:11-22). ExecutionMode is absent: the GPU
    path is deterministic and equals the reference's Sequential mode."""
    grid: GridSpec
    camera: CameraModel = field(default_factory=CameraModel)
    vox_inf: int = 2
    depth: float = 6.5
    tracer_mode: int = N.TRACER_BUNDLED

    def to_c(self) -> N.ConfigC:
        return N.ConfigC(self.grid.c, self.camera.to_c(), self.vox_inf, self.tracer_mode, self.depth)


def bundle_dimensions(cam: CameraModel, depth: float, vox_size: float):
    out = (C.c_int32 * 3)()
    N.check(N.load().vxm_bundle_dimensions(C.byref(cam.to_c()), depth, vox_size, out))
    return tuple(out)


def stats_dict(s: N.StatsC) -> dict:
    d = {k: getattr(s, k) for k, _ in N.StatsC._fields_}
    d["shift_offset"] = tuple(s.shift_offset)
    d["origin"] = tuple(s.origin)
    d["shifted"] = bool(s.shifted)
    return d


class MappingPipeline:
    """MappingPipeline (pipeline.hpp:50-74) for `n_streams` independent sensor
    streams sharing one configuration; every integrate call advances all of
    them by `frames_per_call` consecutive frames on one GPU (frames, poses and
    stats stream-major: frame k of stream s at s*frames_per_call + k)."""

    def __init__(self, cfg: PipelineConfig, initial_position=None, n_streams=1, device=0, flags=0,
                 frames_per_call=1):
        if initial_position is not None:
            g = cfg.grid.c
            cfg = PipelineConfig(GridSpec.create_centered(g.size[0], g.size[1], g.size[2], g.vox_size,
                                                          initial_position),
                                 cfg.camera, cfg.vox_inf, cfg.depth, cfg.tracer_mode)
        self.cfg = cfg
        self.n_streams = n_streams
        self.frames_per_call = frames_per_call
        self.n_slots = n_streams * frames_per_call
        self._lib = N.load()
        self._ctx = C.c_void_p()
        N.check(self._lib.vxm_create_multi(C.byref(cfg.to_c()), n_streams, frames_per_call, device, flags,
                                           C.byref(self._ctx)))
        self._stats = (N.StatsC * self.n_slots)()
        self._poses = (N.PoseC * self.n_slots)()

    def close(self):
        if self._ctx:
            self._lib.vxm_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _set_poses(self, poses):
        """poses: a list of (R, t), or an (n, 12) float64 array (pose_array)."""
        if isinstance(poses, np.ndarray):
            if poses.shape != (self.n_slots, 12) or poses.dtype != np.float64:
                raise ValueError("pose array must be float64 of shape (n_slots, 12)")
            C.memmove(self._poses, np.ascontiguousarray(poses).ctypes.data, poses.nbytes)
            return
        if len(poses) != self.n_slots:
            raise ValueError("need one pose per stream and frame")
        for i, p in enumerate(poses):
            self._poses[i] = pose_c(p)

    def integrate_depth(self, depth, poses):
        """depth: float32 array (S, H, W) or (H, W) in host memory."""
        depth = np.ascontiguousarray(depth, dtype=np.float32)
        cam = self.cfg.camera
        if depth.size != self.n_slots * cam.width * cam.height:
            raise ValueError("depth buffer size does not match camera model")
        if self.n_slots == 1 and not isinstance(poses, list):
            poses = [poses]
        self._set_poses(poses)
        N.check(self._lib.vxm_integrate_depth(self._ctx, C.c_void_p(depth.ctypes.data), self._poses,
                                              self._stats))
        out = [stats_dict(s) for s in self._stats]
        return out[0] if self.n_slots == 1 else out

    def integrate_depth_frames(self, depth, poses):
        """Single-stream contexts: 1..frames_per_call consecutive host frames
        (n, H, W) with n poses; returns n stats dicts (synchronous)."""
        depth = np.ascontiguousarray(depth, dtype=np.float32)
        cam = self.cfg.camera
        n = len(poses)
        if depth.size != n * cam.width * cam.height:
            raise ValueError("depth buffer size does not match camera model")
        pa = (N.PoseC * max(1, n))(*(pose_c(p) for p in poses))
        st = (N.StatsC * max(1, n))()
        N.check(self._lib.vxm_integrate_depth_frames(self._ctx, C.c_void_p(depth.ctypes.data), pa, n, st))
        return [stats_dict(st[i]) for i in range(n)]

    def integrate_depth_frames_ptr(self, depth_ptr: int, poses):
        """integrate_depth_frames from a raw host pointer (e.g. pinned memory,
        which the copy engine reads asynchronously)."""
        n = len(poses)
        pa = (N.PoseC * max(1, n))(*(pose_c(p) for p in poses))
        st = (N.StatsC * max(1, n))()
        N.check(self._lib.vxm_integrate_depth_frames(self._ctx, C.c_void_p(depth_ptr), pa, n, st))
        return [stats_dict(st[i]) for i in range(n)]

    def integrate_depth_ptr(self, depth_ptr: int, poses):
        """Host-buffer entry point for a raw (e.g. pinned) pointer."""
        self._set_poses(poses)
        N.check(self._lib.vxm_integrate_depth(self._ctx, C.c_void_p(depth_ptr), self._poses, self._stats))

    def integrate_depth_device(self, depth_dev_ptr: int, poses):
        """Device-resident frames (n_streams*H*W floats); asynchronous."""
        self._set_poses(poses)
        N.check(self._lib.vxm_integrate_depth_device(self._ctx, C.c_void_p(depth_dev_ptr), self._poses))

    def integrate_depth_async(self, depth_host_ptr: int, poses):
        """Host frames at a raw (pinned) pointer; asynchronous, double
        buffered (H2D of the next call overlaps this call's kernels)."""
        self._set_poses(poses)
        N.check(self._lib.vxm_integrate_depth_async(self._ctx, C.c_void_p(depth_host_ptr), self._poses))

    def wait_stats(self):
        N.check(self._lib.vxm_wait_stats(self._ctx, self._stats))
        return [stats_dict(s) for s in self._stats]

    def integrate(self, xs, ys, zs, t_wc):
        """integrate(MeasurementFrame{cloud, t_wc}) for a camera-frame cloud."""
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        ys = np.ascontiguousarray(ys, dtype=np.float64)
        zs = np.ascontiguousarray(zs, dtype=np.float64)
        self._poses[0] = pose_c(t_wc)
        N.check(self._lib.vxm_integrate_cloud(self._ctx, _f64(xs), _f64(ys), _f64(zs), len(xs),
                                              self._poses, self._stats))
        return stats_dict(self._stats[0])

    def local_grid(self, s=0):
        """(cells uint8[N], origin float64[3]) of stream s."""
        cells = np.empty(self.cfg.grid.cell_count(), dtype=np.uint8)
        origin = np.empty(3, dtype=np.float64)
        N.check(self._lib.vxm_download_local(self._ctx, s, _u8(cells), _f64(origin)))
        return cells, origin

    def set_local_grid(self, cells, origin, s=0):
        cells = np.ascontiguousarray(cells, dtype=np.uint8)
        origin = np.ascontiguousarray(origin, dtype=np.float64)
        N.check(self._lib.vxm_upload_local(self._ctx, s, _u8(cells), _f64(origin)))

    def save_snapshot(self, path, s=0):
        """Checkpoint stream s's local grid as a VOXGRID1 file (grid_io.cpp:14-29)."""
        N.check(self._lib.vxm_snapshot_save(self._ctx, s, str(path).encode()))

    def save_snapshot_async(self, path, s=0):
        """Asynchronous checkpoint (vxm_snapshot_save_async): returns at once;
        later integrate calls proceed; snapshot_wait() joins the file write."""
        N.check(self._lib.vxm_snapshot_save_async(self._ctx, s, str(path).encode()))

    def snapshot_wait(self):
        N.check(self._lib.vxm_snapshot_wait(self._ctx))

    def load_snapshot(self, path, s=0):
        """Resume stream s from a VOXGRID1 file of the same grid layout."""
        N.check(self._lib.vxm_snapshot_load(self._ctx, s, str(path).encode()))

    def set_origin(self, origin, s=0):
        """Places stream s's (empty) local grid, e.g. centred on that stream's
        first camera position (pipeline.hpp:63)."""
        origin = np.ascontiguousarray(origin, dtype=np.float64)
        N.check(self._lib.vxm_upload_local(self._ctx, s, None, _f64(origin)))

    def set_stage_events(self, events):
        """events: 4 cudaEvent_t handles (ints) recorded at the stage
        boundaries of following frames, or None to restore the context's."""
        arr = (C.c_void_p * 4)(*(events or [None] * 4))
        N.check(self._lib.vxm_set_stage_events(self._ctx, arr if events else None))

    def set_input_event(self, event):
        """The next integrate call's kernels wait for this cudaEvent_t (an
        int handle, e.g. torch.cuda.Event.cuda_event) recorded after the
        device frames were produced on another stream."""
        N.check(self._lib.vxm_set_input_event(self._ctx, C.c_void_p(event)))

    def last_frame_ms(self):
        v = C.c_float()
        N.check(self._lib.vxm_last_frame_ms(self._ctx, C.byref(v)))
        return v.value

    @property
    def graph_branches(self) -> int:
        return self._lib.vxm_graph_branches(self._ctx)

    @property
    def cuda_stream(self) -> int:
        return self._lib.vxm_cuda_stream(self._ctx) or 0


# --- synthetic frames on the GPU (sim::render_depth, render.cpp:26-58) -----------

def render_depth(cam: "CameraModel", poses, boxes, out_ptr=None, device=0):
    """Depth frames of an AABB scene for a list of (R, t) camera->world poses.
    boxes: (n, 6) min/max corners. Returns (n_frames, H, W) float32 on the
    host, or renders into a device buffer at out_ptr (n_frames*H*W floats)."""
    boxes = np.ascontiguousarray(boxes, dtype=np.float64).reshape(-1, 6)
    n = len(poses)
    pa = (N.PoseC * n)(*(pose_c(p) for p in poses))
    if out_ptr is None:
        out = np.empty((n, cam.height, cam.width), dtype=np.float32)
        ptr = out.ctypes.data
    else:
        out, ptr = None, out_ptr
    N.check(N.load().vxm_render_depth(C.byref(cam.to_c()), pa, n, boxes.ctypes.data if len(boxes) else None,
                                      len(boxes), C.c_void_p(ptr), device))
    return out


# --- VOXGRID1 dumps (proj/include/voxmap/grid_io.hpp:10-17), host only ----------

def write_grid(grid: "GridSpec", cells, path):
    cells = np.ascontiguousarray(cells, dtype=np.uint8)
    if cells.size != grid.cell_count():
        raise ValueError("write_grid: cell count does not match the grid")
    N.check(N.load().vxm_grid_write(str(path).encode(), C.byref(grid.c), _u8(cells)))


def read_grid(path):
    """-> (GridSpec, cells uint8[N])"""
    spec = N.GridSpecC()
    lib = N.load()
    N.check(lib.vxm_grid_read(str(path).encode(), C.byref(spec), None, 0))
    cells = np.empty(spec.dims[0] * spec.dims[1] * spec.dims[2], dtype=np.uint8)
    N.check(lib.vxm_grid_read(str(path).encode(), C.byref(spec), _u8(cells), cells.size))
    return GridSpec(spec), cells


# --- free functions (stage entry points on host grids) --------------------------

def populate_occupied(grid: GridSpec, ms, xs, ys, zs, t_vc, vox_inf):
    """populate_occupied (integrator.hpp:29-31); ms is updated in place."""
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    st = N.PopulateStatsC()
    N.check(N.load().vxm_populate_occupied(C.byref(grid.c), _u8(ms), _f64(xs), _f64(ys), _f64(zs),
                                           len(xs), C.byref(pose_c(t_vc)), vox_inf, C.byref(st)))
    return {"points_total": st.points_total, "points_outside": st.points_outside}


def _trace_dict(st):
    return {k: getattr(st, k) for k, _ in N.TraceStatsC._fields_}


def trace_bundle(grid: GridSpec, ms, bundle, t_vc, vox_size=None):
    """trace_bundle (raytracer.hpp:130-132), Sequential semantics; vox_size
    defaults to the grid's."""
    b = np.asarray(bundle, dtype=np.int32)
    st = N.TraceStatsC()
    vs = grid.vox_size if vox_size is None else vox_size
    N.check(N.load().vxm_trace_bundle(C.byref(grid.c), _u8(ms), _i32(b), C.byref(pose_c(t_vc)), vs,
                                      C.byref(st)))
    return _trace_dict(st)


def bresenham_trace_image(grid: GridSpec, ms, xs, ys, zs, t_vc):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    st = N.TraceStatsC()
    N.check(N.load().vxm_trace_per_pixel(C.byref(grid.c), _u8(ms), _f64(xs), _f64(ys), _f64(zs), len(xs),
                                         C.byref(pose_c(t_vc)), C.byref(st)))
    return _trace_dict(st)


def merge_grids(local, measurement):
    if local.size != measurement.size:
        raise ValueError("merge_grids: grid layouts differ")
    N.check(N.load().vxm_merge_grids(_u8(local), _u8(measurement), local.size))


def shift_grid_by(dims, cells, offset):
    d = np.asarray(dims, dtype=np.int32)
    o = np.asarray(offset, dtype=np.int32)
    out = np.empty_like(cells)
    N.check(N.load().vxm_shift_grid(_i32(d), _u8(cells), _u8(out), _i32(o)))
    return out


def depth_to_cloud(depth, cam: CameraModel):
    depth = np.ascontiguousarray(depth, dtype=np.float32)
    if depth.size != cam.width * cam.height:
        raise ValueError("depth_to_cloud: image size does not match camera model")
    n = depth.size
    xs, ys, zs = (np.empty(n, dtype=np.float64) for _ in range(3))
    cnt = C.c_size_t()
    N.check(N.load().vxm_depth_to_cloud(C.byref(cam.to_c()), depth.ctypes.data_as(C.POINTER(C.c_float)),
                                        _f64(xs), _f64(ys), _f64(zs), C.byref(cnt)))
    k = cnt.value
    return xs[:k].copy(), ys[:k].copy(), zs[:k].copy()


# --- KernelTable adapter (kernels.hpp:8-33) -------------------------------------

def kernel_merge(local, measurement):
    N.load().vxm_kernel_merge(_u8(local), _u8(measurement), local.size)


def kernel_transform_voxelize(xs, ys, zs, rotation_rowmajor, translation, vox_size):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    R = np.ascontiguousarray(rotation_rowmajor, dtype=np.float64).reshape(9)
    t = np.ascontiguousarray(translation, dtype=np.float64).reshape(3)
    n = len(xs)
    cx, cy, cz = (np.empty(n, dtype=np.int32) for _ in range(3))
    N.load().vxm_kernel_transform_voxelize(_f64(xs), _f64(ys), _f64(zs), n, _f64(R), _f64(t), vox_size,
                                           _i32(cx), _i32(cy), _i32(cz))
    return cx, cy, cz


def kernel_isa() -> str:
    return N.load().vxm_kernel_isa().decode()
