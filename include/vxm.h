/*
 * vxm.h — the C-ABI between the voxmap host library (C++, include/voxmap/)
 * and the hand-written sm_100a kernels in paper_2112_13169_b200/csrc/.
 *
 * Plain C: pointers, sizes and PODs only; no torch or C++ types; no C++
 * exceptions cross it. Every entry point that can fail returns an int status
 * (VXM_OK == 0); the message is available from vxm_last_error() (per calling
 * thread). The C++ wrapper rethrows VXM_EINVAL as std::invalid_argument, like
 * the reference, and everything else as std::runtime_error.
 *
 * The reference interfaces each group replaces are cited next to it
 * (paths relative to /root/reference).
 *
 * Threading: a vxm_ctx owns one cudaStream_t, its device buffers and a
 * captured CUDA graph per frame shape; one caller at a time per context
 * (proj/include/voxmap/pipeline.hpp:50-74 has the same single-caller rule,
 * SPEC.md:387). Distinct contexts are independent and may be driven from
 * different host threads / GPUs concurrently.
 */
#ifndef VXM_H_
#define VXM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VXM_ABI_VERSION 1

enum vxm_status {
  VXM_OK = 0,
  VXM_EINVAL = 1,   /* precondition violated (reference: std::invalid_argument) */
  VXM_ECUDA = 2,    /* CUDA runtime / launch failure */
  VXM_ENOMEM = 3,   /* device or pinned host allocation failed */
  VXM_ENODEV = 4,   /* no sm_100 device visible */
  VXM_ESTATE = 5,   /* call not valid in the context's current state */
  VXM_EIO = 6       /* file I/O or format error (reference: std::runtime_error) */
};

/* Voxel states, one byte per cell (proj/include/voxmap/voxel_state.hpp:9-17). */
enum vxm_voxel_state {
  VXM_UNKNOWN = 0,
  VXM_FREE = 1,
  VXM_OCCUPIED = 2,
  VXM_UNKNOWN_TRACED = 3
};

/* Which tracer frees space (proj/include/voxmap/exec.hpp:13-16). */
enum vxm_tracer_mode { VXM_TRACER_BUNDLED = 0, VXM_TRACER_PER_PIXEL = 1 };

/* GridSpec (proj/include/voxmap/grid.hpp:27-35). Cells are stored flat,
 * idx = x + y*dims[0] + z*dims[0]*dims[1] (grid.hpp:72-77). */
typedef struct vxm_grid_spec {
  double size[3];   /* grid_size_x/y/z, meters */
  double vox_size;  /* meters */
  int32_t dims[3];  /* lround(size / vox_size) per axis */
  int32_t pad_;
  double origin[3]; /* world position of the minimum corner */
} vxm_grid_spec;

/* CameraModel (proj/include/voxmap/geometry.hpp:60-72). */
typedef struct vxm_camera {
  double fov_x;     /* radians */
  double fov_y;     /* radians */
  int32_t width;
  int32_t height;
  double max_depth; /* meters */
} vxm_camera;

/* PipelineConfig (proj/include/voxmap/pipeline.hpp:11-22). ExecutionMode is
 * not carried: the GPU path is always deterministic and equals the
 * reference's Sequential mode bit for bit. */
typedef struct vxm_config {
  vxm_grid_spec grid;
  vxm_camera camera;
  int32_t vox_inf;      /* IntegratorConfig::vox_inf */
  int32_t tracer_mode;  /* enum vxm_tracer_mode */
  double depth;         /* clearing range, meters */
} vxm_config;

/* RigidTransform (geometry.hpp:16-40): p' = R p + t, R row-major. */
typedef struct vxm_pose {
  double rotation[9];
  double translation[3];
} vxm_pose;

/* PipelineStats + TraceStats + PopulateStats (pipeline.hpp:30-41,
 * raytracer.hpp:44-57, integrator.hpp:18-21). The *_us fields are device
 * times of the stages from CUDA events recorded at the stage boundaries
 * when the context records them (VXM_FLAG_STAGE_EVENTS, VXM_FLAG_STAGE_TIMING
 * or VXM_FLAG_NO_GRAPH), else 0; populate_us includes the dilation; shift_us
 * is 0 because the shift is fused into the merge kernel. */
typedef struct vxm_stats {
  uint64_t points_total;
  uint64_t points_outside;
  uint64_t rays_traced;
  uint64_t voxels_freed;
  uint64_t voxels_marked_unknown_traced;
  uint64_t voxels_skipped_out_of_bounds;
  uint64_t occupied_count;
  uint64_t freed_count;
  int32_t shifted;
  int32_t shift_offset[3];
  double origin[3];  /* local-grid origin after this frame */
  double populate_us, trace_us, merge_us, shift_us;
} vxm_stats;

/* ------------------------------------------------------------------------ */
/* Host-side helpers (pure host arithmetic, same formulas as the reference). */

/* GridSpec::create / create_centered (proj/src/grid.cpp:17-52). */
int vxm_grid_spec_create(double size_x, double size_y, double size_z, double vox_size,
                         const double origin[3], vxm_grid_spec* out);
int vxm_grid_spec_create_centered(double size_x, double size_y, double size_z,
                                  double vox_size, const double center[3],
                                  vxm_grid_spec* out);
/* bundle_dimensions (proj/src/raytracer.cpp:8-21): out = {vox_depth, vox_width, vox_height}. */
int vxm_bundle_dimensions(const vxm_camera* cam, double depth, double vox_size,
                          int32_t out[3]);

/* Thread-local message of the last failing call on this thread. */
const char* vxm_last_error(void);
/* "cuda-sm100a" plus build info. */
const char* vxm_build_info(void);
/* Number of visible CUDA devices of compute capability 10.x (0 when none). */
int vxm_device_count(void);

/* ------------------------------------------------------------------------ */
/* Per-stream mapping contexts: MappingPipeline (pipeline.hpp:50-74;
 * proj/src/pipeline.cpp:68-117) for n_streams independent sensor streams
 * that share one configuration, processed as one batch per call.
 * n_streams == 1 is the plain MappingPipeline. */

typedef struct vxm_ctx vxm_ctx;

#define VXM_FLAG_STAGE_TIMING 1u  /* launch stages directly (no graph), events between them */
#define VXM_FLAG_NO_GRAPH 2u      /* launch kernels directly instead of a CUDA graph */
#define VXM_FLAG_SINGLE_BRANCH 4u /* batches: one graph branch (stage events then time each whole stage) */
#define VXM_FLAG_NO_TMA_MERGE 8u  /* K4 with direct loads instead of TMA-staged rows (A/B and fallback) */
#define VXM_FLAG_NO_DESYNC 32u   /* batches: one graph with joined branches instead of per-branch graphs (A/B) */
#define VXM_FLAG_CLEAR_KEYS 64u  /* the large-bundle key format (no epochs, keys reset by the merge) for any
                                    bundle (A/B, tests; chosen anyway above 131,070 rays) */
#define VXM_FLAG_STAGE_EVENTS 16u /* record the stage-boundary events inside the frame graph (fills
                                     vxm_stats::*_us; each event node costs a few us per frame) */

/* cfg->grid must already be placed (use vxm_grid_spec_create_centered to
 * centre it on the first camera position, pipeline.cpp:71-72). Validates as
 * PipelineConfig::validate (pipeline.cpp:33-42). */
int vxm_create(const vxm_config* cfg, int32_t n_streams, int32_t device, uint32_t flags,
               vxm_ctx** out);
/* Multi-frame pipelining (no reference counterpart; SURVEY.md §8f "next" #1):
 * each call takes frames_per_call (F, 1..64) CONSECUTIVE frames of every
 * stream, stream-major (frame k of stream s at index s*F + k, for depth
 * frames, poses and stats alike). Results equal F successive integrate
 * calls bit for bit: the measurement grid origins depend only on the poses
 * (pipeline.cpp:84,102-112), so populate and the ray casts of all F frames
 * run as independent slots, and one chain kernel folds the F merges and
 * shifts in order, producing every frame's counts. vxm_create == F = 1. */
int vxm_create_multi(const vxm_config* cfg, int32_t n_streams, int32_t frames_per_call,
                     int32_t device, uint32_t flags, vxm_ctx** out);
int vxm_destroy(vxm_ctx* ctx);
int vxm_num_streams(const vxm_ctx* ctx);
int vxm_frames_per_call(const vxm_ctx* ctx);
/* Graph branches a batch frame runs as (their kernels overlap on the GPU). */
int vxm_graph_branches(const vxm_ctx* ctx);

/* MappingPipeline::integrate for a depth frame:
 * integrate(MeasurementFrame{depth_to_cloud(img, cam), t_wc}) with the
 * back-projection fused into the first kernel (geometry.cpp:43-99).
 * depth: n_streams * width * height floats, HOST memory, row-major per frame.
 * poses: n_streams camera->world transforms. stats: n_streams outputs.
 * Synchronous: copies in, runs, copies the stats back. */
int vxm_integrate_depth(vxm_ctx* ctx, const float* depth, const vxm_pose* t_wc,
                        vxm_stats* stats);

/* Single-stream contexts: n_frames (1..frames_per_call) consecutive HOST depth
 * frames with their poses, synchronous; n_frames stats. Equals n_frames
 * successive vxm_integrate_depth calls on a single-frame context. */
int vxm_integrate_depth_frames(vxm_ctx* ctx, const float* depth, const vxm_pose* t_wc,
                               int32_t n_frames, vxm_stats* stats);
/* Same, with the depth frames already in device memory (n_streams*W*H
 * floats). Asynchronous: returns after enqueueing; read the stats with
 * vxm_wait_stats(). Batches run on internal streams that the context stream
 * joins, so work the caller enqueues on vxm_cuda_stream() afterwards is
 * ordered after the call; the frames themselves must be complete when the
 * call is made, or signalled by an event passed to vxm_set_input_event. */
int vxm_integrate_depth_device(vxm_ctx* ctx, const float* depth_dev, const vxm_pose* t_wc);
/* The next integrate call's kernels wait for this cudaEvent_t (recorded by
 * the caller after producing the device frames on any stream). One call. */
int vxm_set_input_event(vxm_ctx* ctx, void* cuda_event);
int vxm_wait_stats(vxm_ctx* ctx, vxm_stats* stats);

/* Host frames (pinned for full overlap), asynchronous: the H2D copy runs on a
 * copy stream into one of two device staging buffers, so consecutive calls
 * overlap frame k+1's transfer with frame k's kernels. The host buffer must
 * stay valid until the following vxm_wait_stats (or the next-but-one call). */
int vxm_integrate_depth_async(vxm_ctx* ctx, const float* depth, const vxm_pose* t_wc);

/* MappingPipeline::integrate(MeasurementFrame{cloud, t_wc}) for n_streams == 1
 * with an arbitrary camera-frame point cloud (double SoA, HOST memory). */
int vxm_integrate_cloud(vxm_ctx* ctx, const double* xs, const double* ys, const double* zs,
                        size_t n, const vxm_pose* t_wc, vxm_stats* stats);

/* local_grid() (pipeline.hpp:67): copies stream `s`'s local grid (cell_count
 * bytes) and its origin to HOST memory. */
int vxm_download_local(vxm_ctx* ctx, int32_t s, uint8_t* cells, double origin[3]);
/* Restores stream `s`'s local grid (checkpoint/resume, grid_io.cpp:14-63). */
int vxm_upload_local(vxm_ctx* ctx, int32_t s, const uint8_t* cells, const double origin[3]);

/* VOXGRID1 grid dumps, the reference's snapshot format
 * (proj/include/voxmap/grid_io.hpp:10-17, proj/src/grid_io.cpp:14-69): text
 * header (magic, dims, vox_size, origin with 17 significant digits) then one
 * state byte per cell. vxm_grid_read fills *spec (size = dims * vox_size) and,
 * when cells != NULL, copies the cells (capacity >= cell count). Host only,
 * no GPU needed. VXM_EIO for I/O or format errors. */
int vxm_grid_write(const char* path, const vxm_grid_spec* spec, const uint8_t* cells);
int vxm_grid_read(const char* path, vxm_grid_spec* spec, uint8_t* cells, size_t capacity);
/* Checkpoint / resume of stream s's local grid (cells + origin) through a
 * VOXGRID1 file; the file's dims and vox_size must match the context. */
int vxm_snapshot_save(vxm_ctx* ctx, int32_t s, const char* path);
int vxm_snapshot_load(vxm_ctx* ctx, int32_t s, const char* path);
/* Asynchronous checkpoint: the local grid as it stands
 * after the calls issued so far is copied device -> pinned host memory on a
 * side stream (no context synchronisation; later integrate calls only wait
 * for that ~0.5 MB copy, not for the host) and a host thread writes the
 * VOXGRID1 file (byte-identical to vxm_snapshot_save). One snapshot in
 * flight per context: a new one first waits for the previous.
 * vxm_snapshot_wait joins the writer and returns its status (VXM_EIO on a
 * failed write; VXM_OK when nothing is pending). */
int vxm_snapshot_save_async(vxm_ctx* ctx, int32_t s, const char* path);
int vxm_snapshot_wait(vxm_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) and the device time of the last
 * integrate call's kernels in milliseconds (CUDA events on that stream). */
void* vxm_cuda_stream(vxm_ctx* ctx);
int vxm_last_frame_ms(vxm_ctx* ctx, float* ms);

/* Records the four stage-boundary events inside every following frame into
 * the caller's events (cudaEvent_t: before populate, before trace, after
 * trace, after merge), so per-kernel device times can be read for many
 * queued frames without synchronizing; NULL stops (the context's own events
 * fill vxm_stats::*_us when VXM_FLAG_STAGE_EVENTS is set). */
int vxm_set_stage_events(vxm_ctx* ctx, void* const events[4]);

/* ------------------------------------------------------------------------ */
/* Stage entry points on HOST grids (the free functions of the public API).
 * Each uploads, runs the same kernels as the pipeline, and downloads. */

typedef struct vxm_populate_stats { uint64_t points_total, points_outside; } vxm_populate_stats;
typedef struct vxm_trace_stats {
  uint64_t rays_traced, voxels_freed, voxels_marked_unknown_traced,
      voxels_skipped_out_of_bounds;
} vxm_trace_stats;

/* populate_occupied (proj/include/voxmap/integrator.hpp:29-31,
 * proj/src/integrator.cpp:45-103). ms: cell_count bytes, updated in place. */
int vxm_populate_occupied(const vxm_grid_spec* grid, uint8_t* ms, const double* xs,
                          const double* ys, const double* zs, size_t n,
                          const vxm_pose* t_vc, int32_t vox_inf, vxm_populate_stats* st);

/* trace_bundle (proj/include/voxmap/raytracer.hpp:127-132,
 * proj/src/raytracer.cpp:98-118), Sequential semantics. bundle = {vd, vw, vh};
 * ray_vox_size is trace_bundle's vox_size argument (ray directions and
 * lengths), the walk uses grid->vox_size, as the reference does. */
int vxm_trace_bundle(const vxm_grid_spec* grid, uint8_t* ms, const int32_t bundle[3],
                     const vxm_pose* t_vc, double ray_vox_size, vxm_trace_stats* st);

/* bresenham_trace_image (raytracer.hpp:196-202, raytracer.cpp:120-161), Sequential
 * semantics (last writer in point order wins). */
int vxm_trace_per_pixel(const vxm_grid_spec* grid, uint8_t* ms, const double* xs,
                        const double* ys, const double* zs, size_t n, const vxm_pose* t_vc,
                        vxm_trace_stats* st);

/* merge_grids (proj/include/voxmap/pipeline.hpp:47-48, pipeline.cpp:44-61). */
int vxm_merge_grids(uint8_t* local, const uint8_t* measurement, size_t n);

/* shift_grid_by (proj/include/voxmap/grid.hpp:133, proj/src/grid.cpp:81-108):
 * out[c] = in[c + offset] when in bounds, else Unknown. */
int vxm_shift_grid(const int32_t dims[3], const uint8_t* in, uint8_t* out,
                   const int32_t offset[3]);

/* depth_to_cloud (proj/include/voxmap/geometry.hpp:131-132,
 * proj/src/geometry.cpp:64-99): row-major compaction of valid pixels.
 * xs/ys/zs must hold width*height doubles; *n_out receives the point count. */
int vxm_depth_to_cloud(const vxm_camera* cam, const float* depth, double* xs, double* ys,
                       double* zs, size_t* n_out);

/* sim::render_depth (proj/include/voxmap/sim/render.hpp:11-20,
 * proj/src/sim/render.cpp:8-58): synthetic depth frames of an AABB scene
 * (boxes: n_boxes x {min_x, min_y, min_z, max_x, max_y, max_z}) from n_frames
 * camera->world poses, bit-identical to the reference renderer. out: HOST or
 * DEVICE memory (on `device`), n_frames * width * height floats (0 = no
 * return within max_depth). Input generation for large batches. */
int vxm_render_depth(const vxm_camera* cam, const vxm_pose* t_wc, int32_t n_frames,
                     const double* boxes, int32_t n_boxes, float* out, int32_t device);
/* ------------------------------------------------------------------------ */
/* KernelTable adapter (proj/include/voxmap/kernels/kernels.hpp:8-33): the
 * exact MergeFn / TransformVoxelizeFn signatures, HOST pointers, void, no
 * allocation visible to the caller, any alignment, any n (including 0).
 * Errors abort with a message: the reference signature has no error channel.
 * Useful for parity (each call pays H2D + D2H). */
void vxm_kernel_merge(uint8_t* local, const uint8_t* measurement, size_t n);
void vxm_kernel_transform_voxelize(const double* xs, const double* ys, const double* zs,
                                   size_t n, const double* rotation,
                                   const double* translation, double vox_size, int32_t* cx,
                                   int32_t* cy, int32_t* cz);
const char* vxm_kernel_isa(void); /* "cuda-sm100a" */

#ifdef __cplusplus
}
#endif

#endif /* VXM_H_ */
