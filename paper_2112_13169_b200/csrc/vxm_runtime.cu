// C-ABI runtime (include/vxm.h): per-stream mapping contexts, the per-frame
// CUDA graph, and the stand-alone stage entry points.
//
// Per-frame flow for a context of S streams (MappingPipeline::integrate,
// proj/src/pipeline.cpp:74-117, batched over streams):
//   host:  validate t_wc, T_vc = compose(T(-origin), t_wc), shift decision,
//          epoch bump -> FrameParams[S] in pinned memory
//   H2D:   FrameParams (and the depth frames for the host-buffer entry point)
//   graph: K1 populate | K2 dilate (vox_inf > 0) | K3 trace_bundle |
//          K4 merge+shift+count | K5 publish (counters to host-mapped
//          memory, cleared for the next frame)
// Batches of >= 12 slots run as three branches over shares of the streams;
// for single-frame batches each branch is its own graph on its own stream,
// waiting only for its call's inputs, and the context stream joins them
// (run_frame). The measurement grid is never reset: epoch-tagged words
// (vxm_device.cuh).

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vxm.h"
#include "host/voxgrid_format.hpp"
#include "vxm_aux_kernels.cuh"
#include "vxm_kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct CudaError {
  int code;
};

#define VXM_CK(call)                                                                      \
  do {                                                                                    \
    const cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                              \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                         \
      throw CudaError{e_ == cudaErrorMemoryAllocation ? VXM_ENOMEM : VXM_ECUDA};          \
    }                                                                                     \
  } while (0)

struct InvalidArg {
  std::string what;
};

struct IoError {
  std::string what;
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return VXM_OK;
  } catch (const CudaError& e) {
    return e.code;
  } catch (const InvalidArg& e) {
    return fail(VXM_EINVAL, e.what);
  } catch (const IoError& e) {
    return fail(VXM_EIO, e.what);
  } catch (const std::bad_alloc&) {
    return fail(VXM_ENOMEM, "host allocation failed");
  }
}

// ---------------------------------------------------------------------------
// Host arithmetic, operation for operation as the reference.
// ---------------------------------------------------------------------------

// GridSpec::create (proj/src/grid.cpp:17-42).
void spec_create(double sx, double sy, double sz, double vs, const double origin[3],
                 vxm_grid_spec* out) {
  if (!(vs > 0.0)) throw InvalidArg{"vox_size must be positive"};
  if (!(sx > 0.0) || !(sy > 0.0) || !(sz > 0.0)) throw InvalidArg{"grid sizes must be positive"};
  for (int a = 0; a < 3; ++a)
    if (!std::isfinite(origin[a])) throw InvalidArg{"grid origin must be finite"};
  out->size[0] = sx;
  out->size[1] = sy;
  out->size[2] = sz;
  out->vox_size = vs;
  out->dims[0] = static_cast<int>(std::lround(sx / vs));
  out->dims[1] = static_cast<int>(std::lround(sy / vs));
  out->dims[2] = static_cast<int>(std::lround(sz / vs));
  out->pad_ = 0;
  for (int a = 0; a < 3; ++a) out->origin[a] = origin[a];
  if (out->dims[0] < 1 || out->dims[1] < 1 || out->dims[2] < 1)
    throw InvalidArg{"grid must be at least one voxel per axis"};
}

// GridSpec::half_extent (grid.hpp:56-60): integer halving, then * vox_size.
double half_extent(const vxm_grid_spec& g, int a) {
  return static_cast<double>(g.dims[a] / 2) * g.vox_size;
}

// CameraModel::validate (proj/src/geometry.cpp:28-41).
void camera_validate(const vxm_camera& c) {
  if (c.width <= 0 || c.height <= 0)
    throw InvalidArg{"CameraModel: width and height must be positive"};
  const double pi = 3.14159265358979323846;
  if (!(c.fov_x > 0.0) || !(c.fov_x < pi) || !(c.fov_y > 0.0) || !(c.fov_y < pi))
    throw InvalidArg{"CameraModel: FOV must lie in (0, pi)"};
  if (!(c.max_depth > 0.0) || !std::isfinite(c.max_depth))
    throw InvalidArg{"CameraModel: max_depth must be positive and finite"};
}

// bundle_dimensions (proj/src/raytracer.cpp:8-21).
void bundle_dims(const vxm_camera& cam, double depth, double vs, int32_t out[3]) {
  camera_validate(cam);
  if (!(depth > 0.0) || !std::isfinite(depth))
    throw InvalidArg{"bundle_dimensions: depth must be positive and finite"};
  if (!(vs > 0.0) || !std::isfinite(vs))
    throw InvalidArg{"bundle_dimensions: vox_size must be positive and finite"};
  out[0] = std::max(1, static_cast<int>(std::lround(depth / vs)));
  out[1] = 2 * static_cast<int>(std::lround(std::tan(cam.fov_x / 2.0) * out[0])) + 1;
  out[2] = 2 * static_cast<int>(std::lround(std::tan(cam.fov_y / 2.0) * out[0])) + 1;
}

bool all_finite(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// RigidTransform::is_valid (proj/src/geometry.cpp:17-22) with the Eigen
// subset's arithmetic: gram = R^T R (left-to-right dot products), max |gram-I|,
// determinant by cofactors of the first column.
bool pose_valid(const vxm_pose& p, double tol) {
  if (!all_finite(p.rotation, 9) || !all_finite(p.translation, 3)) return false;
  auto R = [&](int i, int j) { return p.rotation[3 * i + j]; };
  double worst = 0.0;
  bool first = true;
  for (int j = 0; j < 3; ++j) {
    for (int i = 0; i < 3; ++i) {
      double acc = R(0, i) * R(0, j);
      acc = acc + R(1, i) * R(1, j);
      acc = acc + R(2, i) * R(2, j);
      double d = acc - (i == j ? 1.0 : 0.0);
      d = d < 0.0 ? -d : d;
      if (first || d > worst) worst = d;
      first = false;
    }
  }
  if (worst > tol) return false;
  const double det = R(0, 0) * (R(1, 1) * R(2, 2) - R(2, 1) * R(1, 2)) -
                     R(1, 0) * (R(0, 1) * R(2, 2) - R(2, 1) * R(0, 2)) +
                     R(2, 0) * (R(0, 1) * R(1, 2) - R(1, 1) * R(0, 2));
  return std::abs(det - 1.0) <= tol;
}

// camera_to_grid_transform = compose(T(-origin), t_wc) (pipeline.cpp:63-66,
// geometry.cpp:24-26): R_vc = I * R_wc, t_vc = I * t_wc + (-origin), each
// product a left-to-right dot product as in the Eigen subset.
void camera_to_grid(const vxm_pose& t_wc, const double origin[3], double rot[9],
                    double trans[3]) {
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) {
      double acc = (i == 0 ? 1.0 : 0.0) * t_wc.rotation[0 * 3 + j];
      acc = acc + (i == 1 ? 1.0 : 0.0) * t_wc.rotation[1 * 3 + j];
      acc = acc + (i == 2 ? 1.0 : 0.0) * t_wc.rotation[2 * 3 + j];
      rot[3 * i + j] = acc;
    }
    double acc = (i == 0 ? 1.0 : 0.0) * t_wc.translation[0];
    acc = acc + (i == 1 ? 1.0 : 0.0) * t_wc.translation[1];
    acc = acc + (i == 2 ? 1.0 : 0.0) * t_wc.translation[2];
    trans[i] = acc + (-origin[i]);
  }
}

// The recentring rule of MappingPipeline::integrate (pipeline.cpp:102-112)
// and shift_offset_for_center (grid.cpp:110-117). Returns true when the grid
// moves; `origin` is updated to the shifted grid's origin (grid.cpp:84).
bool shift_decision(const vxm_grid_spec& g, double origin[3], const double t[3], int32_t off[3]) {
  const double vs = g.vox_size;
  bool drifted = false;
  for (int a = 0; a < 3; ++a) {
    const double center = origin[a] + half_extent(g, a);
    double drift = t[a] - center;
    drift = drift < 0.0 ? -drift : drift;
    if (drift >= vs) drifted = true;
  }
  off[0] = off[1] = off[2] = 0;
  if (!drifted) return false;
  for (int a = 0; a < 3; ++a) {
    const double ideal = t[a] - half_extent(g, a);
    const double delta = (ideal - origin[a]) / vs;
    off[a] = static_cast<int32_t>(std::lround(delta));
  }
  if (off[0] == 0 && off[1] == 0 && off[2] == 0) return false;
  for (int a = 0; a < 3; ++a) origin[a] = origin[a] + static_cast<double>(off[a]) * vs;
  return true;
}

int sm_count(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 148;
}

void check_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    g_err = "no CUDA device visible";
    throw CudaError{VXM_ENODEV};
  }
  if (device < 0 || device >= count) throw InvalidArg{"device index out of range"};
  cudaDeviceProp prop;
  VXM_CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    g_err = std::string("device ") + prop.name + " is not sm_100 (this build targets sm_100a only)";
    throw CudaError{VXM_ENODEV};
  }
}

constexpr int kPopulateThreads = 256;
constexpr int kMergeThreads = 256;

}  // namespace

void vxm_set_error(const char* msg) { g_err = msg ? msg : ""; }

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------
struct vxm_ctx {
  vxm_config cfg{};
  int S = 1;       // independent sensor streams
  int F = 1;       // consecutive frames of each stream per call
  int nslots = 1;  // S * F measurement grids (slot = s * F + k)
  int device = 0;
  uint32_t flags = 0;
  int nsm = 148;
  cudaStream_t stream = nullptr;
  vxm::KParams kp{};
  long long n = 0;
  long long rows = 0;  // x-rows per grid (dy * dz)
  int32_t bundle[3] = {0, 0, 0};

  // device buffers
  uint8_t* occ = nullptr;
  uint8_t* ctr = nullptr;
  uint8_t* rowflag = nullptr;  // per slot: dy*dz x-row flags (vox_inf > 0)
  uint32_t* key = nullptr;     // measurement keys (vxm_device.cuh KeyFmt)
  int key_fmt = vxm::kEpochKeys;
  uint8_t* loc[2] = {nullptr, nullptr};
  double* qtab = nullptr;  // W column + H row back-projection factors
  uint32_t* dbits = nullptr;  // x-dilated centre bit rows (vox_inf > 0)
  uint8_t* dtmp = nullptr;    // generic dilation passes (large radii / rows)
  vxm::Counters* counters = nullptr;
  // FrameParams on the device, two buffers: the upload for the next call
  // (on param_stream) overlaps the graph of this one, and each buffer has
  // its own instance of every frame graph
  static constexpr int kPP = VXM_PP;
  vxm::FrameParams* frames_pp[kPP] = {nullptr, nullptr};
  int pp = 0;  // buffer of the current call
  bool sync_call = false;  // the current call waits for its stats (vxm_integrate_depth / _cloud)
  cudaStream_t param_stream = nullptr;
  cudaEvent_t pp_ready[kPP] = {}, pp_free[kPP] = {};
  float* depth_dev = nullptr;
  // double-buffered staging for vxm_integrate_depth_async (created lazily)
  cudaStream_t copy_stream = nullptr;
  static constexpr int kBranches = VXM_BRANCHES;
  cudaStream_t side[kBranches] = {};  // streams of graph branches 1..
  cudaEvent_t fork[kBranches] = {}, join[kBranches] = {};
  cudaEvent_t chain[kBranches] = {};  // a chained range's merge is done (merge_ranges)
  // desynchronised batches (run_frame): branch b's frame graph runs on its own
  // stream, waiting only for this call's inputs, and the context stream joins
  cudaStream_t dside[kBranches] = {};
  cudaEvent_t ddone[kBranches] = {};
  cudaEvent_t bstart[kBranches] = {};  // a desynchronised branch's start (timing events)
  int desync_started = 0;              // branches whose bstart brackets the last call
  cudaEvent_t input_ready = nullptr;  // set by a call whose inputs arrive on another stream
  cudaEvent_t user_input = nullptr;   // vxm_set_input_event: the next call's kernels wait for it
  // asynchronous snapshot (vxm_snapshot_save_async): D2H of one local grid on
  // snap_stream into pinned snap_host, then a writer thread; the next call's
  // kernels wait for snap_copied (the ping-pong buffer is rewritten two
  // frames later)
  cudaStream_t snap_stream = nullptr;
  cudaEvent_t snap_start = nullptr, snap_copied = nullptr;
  uint8_t* snap_host = nullptr;
  bool snap_wait_pending = false;
  std::thread snap_thread;
  int snap_status = 0;
  std::string snap_error;
  cudaEvent_t tail_ev = nullptr;      // end of the last call that ran on the context stream itself
  bool tail_pending = false;          // ... which desynchronised branches must still wait for
  std::vector<int> wrapped;           // slots whose arrays are cleared before this call (epoch wrap)
  float* stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_copied[2] = {};
  cudaEvent_t ev_consumed[2] = {};
  int stage_slot = 0;
  double* cloud_dev = nullptr;
  size_t cloud_cap = 0;

  // pinned host mirrors; FrameParams go through a ring so that a frame can be
  // prepared while earlier ones are still queued
  static constexpr int kRing = 4;
  vxm::FrameParams* frames_ring = nullptr;  // kRing * S
  cudaEvent_t ring_ev[kRing] = {};
  int ring_slot = 0;
  vxm::FrameParams* frames_host = nullptr;  // current ring slot
  vxm::CountersHead* counters_host = nullptr;  // host-mapped, written by K4

  // host state per stream
  std::vector<uint32_t> epoch;
  std::vector<uint32_t> cur;
  std::vector<double> origin;  // 3 per stream
  std::vector<int32_t> last_off;      // per slot
  std::vector<int32_t> last_shifted;  // per slot
  std::vector<double> origin_after;   // per slot: local origin after that frame

  // captured frame graphs: 0 depth, 1 cloud, 2 depth with the compacting K1
  static constexpr int kGraphs = 3;
  cudaGraphExec_t graph_exec[kGraphs][kPP] = {};
  cudaGraphExec_t bgraph[kGraphs][kPP][kBranches] = {};  // per-branch frame graphs (desynchronised batches)
  cudaGraph_t graph_tmpl[kGraphs][kPP] = {};               // kept for node updates
  cudaGraphNode_t stage_nodes[kGraphs][kPP][4] = {};       // event-record nodes per graph
  bool pop_compact = false;  // K1 variant: valid fraction of the last observed frames < 1/2
  void* user_stage_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool stage_clean[kGraphs][kPP] = {};  // node events point where they should
  bool graph_marks[kGraphs][kPP] = {};  // the instance holds the stage event-record nodes
  bool capture_marks = false;           // capture in progress records them
  bool last_marks = false;              // the last frame recorded them
  // ev[0] / ev[5] bracket the frame outside the graph; ev[1..4] are the
  // stage boundaries recorded inside it (before populate, before trace,
  // after trace, after merge)
  cudaEvent_t ev[6] = {};
  bool pending = false;
  float last_ms = 0.f;
};

namespace {

// capturing: inside stream capture the stage events must be recorded as
// external event-record nodes (a plain record only adds a dependency edge).
int graph_branches(const vxm_ctx* c) {
  const bool single = (c->flags & (VXM_FLAG_STAGE_TIMING | VXM_FLAG_SINGLE_BRANCH)) != 0;
  return !single && c->nslots >= 4 * vxm_ctx::kBranches ? vxm_ctx::kBranches : 1;
}

// A single stream with F > 1 frames per call and graph branches: branch b
// handles the frame range [F*b/B, F*(b+1)/B) and merges it as its own chain
// once the previous range's merge is done, so the chain merges of the early
// ranges overlap the later ranges' populate and trace (measured: +6% for 64
// frames per call; 4% slower for 16, where each range's extra pass over the
// grid costs more than the overlap saves, hence F >= 32). Returns the number
// of chained merges (1 otherwise).
int merge_ranges(const vxm_ctx* c) {
  return c->S == 1 && c->F >= 32 ? graph_branches(c) : 1;
}

// The four stages for slots [s0, s0 + S) on stream `st` (kernel parameters
// rebased to the first slot). `marks` records the stage-boundary events.
bool launch_merge(vxm_ctx* c, const vxm::KParams& kp, int S, cudaStream_t st);

// K5 over S slots: counters -> host-mapped read-back, cleared for the next frame
void launch_publish(const vxm::KParams& kp, int S, cudaStream_t st) {
  VXM_CK(vxm::launch_pdl(vxm::publish_counters_kernel, dim3(S), dim3(128), 0, st, kp));
}

void launch_stages(vxm_ctx* c, bool cloud, bool capturing, int s0, int S, cudaStream_t st, bool marks,
                   bool merge = true) {
  vxm::KParams kp = c->kp;
  const long long n = c->n;
  kp.frames += s0;
  kp.counters += s0;
  kp.counters_out += s0;
  kp.occ += n * s0;
  kp.key += c->n * s0;
  if (kp.ctr) kp.ctr += n * s0;
  if (kp.rowflag) kp.rowflag += c->rows * s0;
  if (kp.dbits) kp.dbits += static_cast<long long>(vxm::dilate_row_words(kp.dx)) * c->rows * s0;
  if (kp.dtmp) kp.dtmp += 2 * n * s0;
  kp.loc0 += n * (s0 / c->F);
  kp.loc1 += n * (s0 / c->F);
  auto mark = [&](cudaEvent_t e) {
    if (!marks) return;
    if (capturing) {  // graph nodes, re-pointed at the caller's events by apply_stage_events
      VXM_CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
      return;
    }
    for (int i = 0; i < 4; ++i)  // direct launches record the caller's events when attached
      if (e == c->ev[1 + i] && c->user_stage_ev[i]) e = static_cast<cudaEvent_t>(c->user_stage_ev[i]);
    VXM_CK(cudaEventRecord(e, st));
  };
  mark(c->ev[1]);
  if (!cloud) {
    // tiles of 256 quads; a block takes `iters` of them once the batch
    // alone fills the GPU several times over (8 blocks per SM)
    const long long npix = static_cast<long long>(kp.W) * kp.H;
    const long long tiles = ((npix + 3) / 4 + kPopulateThreads - 1) / kPopulateThreads;
    const long long fill = static_cast<long long>(c->nsm) * 8;
    // (measured: at least min(4, what the whole call would use) when graph
    // branches launch small shares concurrently: +6% at 16 streams)
    const long long want = std::max(tiles * S / fill, std::min(4LL, tiles * c->nslots / fill));
    const int iters = static_cast<int>(std::max(1LL, std::min<long long>(vxm::kPopMaxIters, want)));
    dim3 grid(static_cast<unsigned>((tiles + iters - 1) / iters), S);
    if (npix % 4 == 0) {
      // staged quads + per-warp lists of valid pixels (u16, 4 per quad)
      const size_t smem = (sizeof(float4) + 4 * sizeof(uint16_t)) * kPopulateThreads * static_cast<size_t>(iters);
      const bool clr = kp.key_fmt == vxm::kClearKeys;
      auto k1 = c->pop_compact ? (clr ? vxm::populate_depth_tma_kernel<true, true> : vxm::populate_depth_tma_kernel<true, false>)
                               : (clr ? vxm::populate_depth_tma_kernel<false, true> : vxm::populate_depth_tma_kernel<false, false>);
      VXM_CK(vxm::launch_ex(false, k1, grid, dim3(kPopulateThreads), smem, st, kp, iters));
    } else {
      VXM_CK(vxm::launch_ex(false,
                            kp.key_fmt == vxm::kClearKeys ? vxm::populate_depth_kernel<true> : vxm::populate_depth_kernel<false>,
                            grid, dim3(kPopulateThreads), 0, st, kp, iters));
    }
  } else {
    dim3 grid(static_cast<unsigned>(c->nsm * 4), S);
    VXM_CK(vxm::launch_ex(false,
                          kp.key_fmt == vxm::kClearKeys ? vxm::populate_cloud_kernel<true> : vxm::populate_cloud_kernel<false>,
                          grid, dim3(kPopulateThreads), 0, st, kp));
  }
  VXM_CK(cudaGetLastError());
  if (kp.vox_inf > 0) {
    const int r = kp.vox_inf;
    vxm::launch_dilate(kp, r, S, vxm::dilate_smem_bytes(r, kp.dx), st);
    VXM_CK(cudaGetLastError());
  }
  mark(c->ev[2]);
  {
    if (c->cfg.tracer_mode == VXM_TRACER_PER_PIXEL) {
      const long long n = cloud ? static_cast<long long>(c->nsm) * 4 * kPopulateThreads
                                : static_cast<long long>(kp.W) * kp.H;
      dim3 grid(static_cast<unsigned>(std::min<long long>((n + 255) / 256, c->nsm * 8)), S);
      VXM_CK(vxm::launch_pdl(vxm::trace_per_pixel_kernel, grid, dim3(256), 0, st, kp, cloud ? 0 : 1));
    } else {
      vxm::launch_trace(kp, S, c->nslots, st);
    }
    VXM_CK(cudaGetLastError());
  }
  mark(c->ev[3]);
  if (merge) {
    if (!launch_merge(c, kp, S, st)) launch_publish(kp, S, st);
  }
  mark(c->ev[4]);
}

// K4 for S slots of rebased parameters: merge + shift + counts (F == 1), or
// the chain kernel over S / F streams (F > 1).
// K4' over `streams` streams of F frames each (kp rebased to the first)
// Returns true: the chain kernel publishes the counters itself (no K5).
bool launch_merge_chain(vxm_ctx* c, const vxm::KParams& kp_in, int F, int streams, cudaStream_t st) {
  vxm::KParams kp = kp_in;
  kp.k4_publish = 1;
  // chains of F frames per stream; the chain box varies per call, so the
  // launch covers it with a fixed grid-stride shape
  const long long chains = c->n * 2;
  constexpr int kChainThreads = VXM_SEQ_THREADS;
  const long long blocks = std::min<long long>((chains + kChainThreads - 1) / kChainThreads,
                                               std::max<long long>(1, c->nsm * (2048LL / kChainThreads) / streams));
  dim3 grid(static_cast<unsigned>(std::max<long long>(1, blocks)), streams);
  if (kp.key_fmt == vxm::kClearKeys)
    VXM_CK(vxm::launch_pdl(vxm::merge_sequence_kernel<true>, grid, dim3(kChainThreads), 0, st, kp, F));
  else
    VXM_CK(vxm::launch_pdl(vxm::merge_sequence_epoch_kernel, grid, dim3(kChainThreads), 0, st, kp, F));
  VXM_CK(cudaGetLastError());
  return true;
}

// Returns true when the K4 launched publishes the counters itself (no K5).
bool launch_merge(vxm_ctx* c, const vxm::KParams& kp, int S, cudaStream_t st) {
  // Short rows whose cells move as words (dx % 4 == 0, dx <= 128: every
  // benchmark grid) take the direct-load K4 with four rows of loads in flight
  // per lane; it measured faster there than the TMA-staged K4 (57 vs 70 us for
  // 64 cfg2 slots). Longer or odd rows take the TMA-staged K4 (57 vs 72 us for
  // 8 cfg3 slots of 200-cell rows).
  const bool direct_vec = kp.dx % 4 == 0 && kp.dx <= VXM_MERGE_DIRECT_MAX_DX;
  if (c->F == 1 && !direct_vec && kp.dx <= vxm::kMergeTmaMaxDx && !(c->flags & VXM_FLAG_NO_TMA_MERGE)) {
    // groups of merge_tma_rows rows; each block pipelines several (two stages)
    const int rows = vxm::merge_tma_rows(kp.dx, kp.dy);
    const long long groups = static_cast<long long>((kp.dy + rows - 1) / rows) * kp.dz;
    const long long per_slot = std::max(1LL, std::min(groups, c->nsm * 8LL / S));
    const dim3 grid(static_cast<unsigned>(per_slot), S);
    const size_t smem = 2 * vxm::merge_tma_smem_bytes(rows * kp.dx);
    if (kp.key_fmt == vxm::kClearKeys)
      VXM_CK(vxm::launch_pdl(vxm::merge_shift_count_tma_kernel<true>, grid, dim3(kMergeThreads), smem, st, kp));
    else
      VXM_CK(vxm::launch_pdl(vxm::merge_epoch_tma_kernel, grid, dim3(kMergeThreads), smem, st, kp));
  } else if (c->F == 1) {
    const long long rows = static_cast<long long>(kp.dy) * kp.dz;
    // one row per warp unless the batch fills the GPU several times over
    const long long warps = rows * c->nslots;  // the whole call (branches run concurrently)
    const long long fill = static_cast<long long>(c->nsm) * 64;
    const long long rpw_max = warps / fill >= VXM_MERGE_RPW ? VXM_MERGE_RPW : vxm::kRowsPerWarp;
    const int rpw = static_cast<int>(std::max<long long>(VXM_MERGE_RPW_MIN, std::min<long long>(rpw_max, warps / fill)));
    const int rows_per_block = kMergeThreads / 32 * rpw;
    dim3 grid(static_cast<unsigned>((rows + rows_per_block - 1) / rows_per_block), S);
    if (kp.key_fmt == vxm::kClearKeys) {
      VXM_CK(vxm::launch_pdl(vxm::merge_shift_count_kernel<true>, grid, dim3(kMergeThreads), 0, st, kp, rpw));
    } else {
      vxm::KParams kq = kp;
      kq.k4_publish = 1;
      VXM_CK(vxm::launch_pdl(vxm::merge_epoch_kernel, grid, dim3(kMergeThreads), 0, st, kq, rpw));
      VXM_CK(cudaGetLastError());
      return true;
    }
    VXM_CK(cudaGetLastError());
  } else {
    return launch_merge_chain(c, kp, c->F, S / c->F, st);
  }
  return false;
}

// One frame of every slot: the stages, optionally as graph branches over
// shares of the streams (kernels of one branch overlap the others'); K4
// then K5 publishes the counters to the host-mapped read-back buffer.
void launch_frame(vxm_ctx* c, bool cloud, bool capturing) {
  // stage-boundary events: always for direct launches (cheap stream
  // records); in a graph only when asked for, since every event-record node
  // splits the graph's execution (measured: 17 us per single-stream frame
  // for five nodes, 0.065 -> 0.048 ms)
  const bool marks = !capturing || c->capture_marks;
  // Batches run as kBranches graph branches over equal shares of the streams:
  // the branches' stages overlap on the GPU (the ALU-bound trace of one share
  // with the HBM-bound populate / merge of another; +13% frames/s at 64
  // streams, tools/quick_time.py). One branch for single streams, F > 1, the
  // stage-timing mode and VXM_FLAG_SINGLE_BRANCH.
  const int B = cloud ? 1 : graph_branches(c);
  if (B > 1) {
    for (int b = 1; b < B; ++b)
      if (!c->side[b]) {
        VXM_CK(cudaStreamCreateWithFlags(&c->side[b], cudaStreamNonBlocking));
        VXM_CK(cudaEventCreateWithFlags(&c->fork[b], cudaEventDisableTiming));
        VXM_CK(cudaEventCreateWithFlags(&c->join[b], cudaEventDisableTiming));
      }
    for (int b = 0; b < B; ++b)
      if (!c->chain[b]) VXM_CK(cudaEventCreateWithFlags(&c->chain[b], cudaEventDisableTiming));
    for (int b = 1; b < B; ++b) {
      VXM_CK(cudaEventRecord(c->fork[b], c->stream));
      VXM_CK(cudaStreamWaitEvent(c->side[b], c->fork[b], 0));
    }
    // At least as many streams as branches: each branch runs all stages for
    // whole streams (all F frames of each, chain merge included). Fewer
    // streams (F > 1): the branches run K1-K3 for shares of the frame slots,
    // then either each merges its frame range as a chain after the previous
    // range (one stream, merge_ranges) or the chain merge of every stream
    // follows once they joined.
    const bool by_stream = c->S >= B;
    const int units = by_stream ? c->S : c->nslots;
    const int per_unit = by_stream ? c->F : 1;  // slots per unit
    const bool chained = !by_stream && merge_ranges(c) > 1;
    for (int b = 0; b < B; ++b) {
      const int s0 = units * b / B * per_unit, s1 = units * (b + 1) / B * per_unit;
      cudaStream_t bs = b == 0 ? c->stream : c->side[b];
      launch_stages(c, cloud, capturing, s0, s1 - s0, bs, b == 0 && marks, by_stream);
      if (chained) {
        // this range's chain merge, after the previous range's
        if (b > 0) VXM_CK(cudaStreamWaitEvent(bs, c->chain[b - 1], 0));
        vxm::KParams kp = c->kp;
        kp.frames += s0;
        kp.counters += s0;
        kp.counters_out += s0;
        kp.occ += c->n * s0;
        kp.key += c->n * s0;
        if (!launch_merge_chain(c, kp, s1 - s0, 1, bs)) launch_publish(kp, s1 - s0, bs);
        if (b + 1 < B) VXM_CK(cudaEventRecord(c->chain[b], bs));
      }
    }
    for (int b = 1; b < B; ++b) {
      VXM_CK(cudaEventRecord(c->join[b], c->side[b]));
      VXM_CK(cudaStreamWaitEvent(c->stream, c->join[b], 0));
    }
    if (!by_stream && !chained) {
      if (!launch_merge(c, c->kp, c->nslots, c->stream)) launch_publish(c->kp, c->nslots, c->stream);
    }
  } else {
    launch_stages(c, cloud, capturing, 0, c->nslots, c->stream, marks);
  }
}

cudaGraphExec_t capture(vxm_ctx* c, bool cloud, int gi, int pp, bool marks) {
  c->capture_marks = marks;
  c->graph_marks[gi][pp] = marks;
  cudaGraph_t g = nullptr;
  VXM_CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    launch_frame(c, cloud, true);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  VXM_CK(cudaStreamEndCapture(c->stream, &g));
  c->graph_tmpl[gi][pp] = g;
  // locate the stage event-record nodes so callers can redirect them
  size_t nn = 0;
  VXM_CK(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  VXM_CK(cudaGraphGetNodes(g, nodes.data(), &nn));
  for (cudaGraphNode_t node : nodes) {
    cudaGraphNodeType type;
    VXM_CK(cudaGraphNodeGetType(node, &type));
    if (type != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t e = nullptr;
    VXM_CK(cudaGraphEventRecordNodeGetEvent(node, &e));
    for (int i = 0; i < 4; ++i)
      if (e == c->ev[1 + i]) c->stage_nodes[gi][pp][i] = node;
  }
  cudaGraphExec_t exec = nullptr;
  VXM_CK(cudaGraphInstantiate(&exec, g, 0));
  return exec;
}

// Points the graph's stage event-record nodes at the caller's events (or
// back at the context's own).
void apply_stage_events(vxm_ctx* c, cudaGraphExec_t exec, int gi, int pp) {
  for (int i = 0; i < 4; ++i) {
    if (!c->stage_nodes[gi][pp][i]) continue;
    cudaEvent_t e = c->user_stage_ev[i] ? static_cast<cudaEvent_t>(c->user_stage_ev[i]) : c->ev[1 + i];
    VXM_CK(cudaGraphExecEventRecordNodeSetEvent(exec, c->stage_nodes[gi][pp][i], e));
  }
}

// Host half of one frame for every stream: validation, T_vc, shift, epoch.
// Claims the next FrameParams ring slot (waiting until the copy that last
// used it has executed).
void next_slot(vxm_ctx* c) {
  c->ring_slot = (c->ring_slot + 1) % vxm_ctx::kRing;
  VXM_CK(cudaEventSynchronize(c->ring_ev[c->ring_slot]));
  c->frames_host = c->frames_ring + static_cast<size_t>(c->ring_slot) * c->nslots;
}

void prepare_frames(vxm_ctx* c, const vxm_pose* poses, const float* depth_dev_base,
                    size_t frame_elems) {
  c->wrapped.clear();
  for (int i = 0; i < c->nslots; ++i) {
    if (!pose_valid(poses[i], 1e-6)) throw InvalidArg{"MeasurementFrame: invalid transform"};
  }
  const int R = merge_ranges(c);
  for (int s = 0; s < c->S; ++s) {
    double* org = &c->origin[3 * s];
    int32_t P[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    int range = 0, k0 = 0;  // chained merge range of frame k and its first frame
    for (int k = 0; k < c->F; ++k) {
      const int slot = s * c->F + k;
      vxm::FrameParams& f = c->frames_host[slot];
      if (R > 1 && k == c->F * (range + 1) / R) {
        // close the previous range's chain box (relative to its first frame)
        vxm::FrameParams& fr = c->frames_host[s * c->F + k0];
        for (int a = 0; a < 3; ++a) {
          fr.box_lo[a] = lo[a];
          fr.box_ext[a] = hi[a] - lo[a] + c->cfg.grid.dims[a];
          P[a] = lo[a] = hi[a] = 0;
        }
        ++range;
        k0 = k;
      }
      // the measurement grid takes the local grid's pre-shift origin (pipeline.cpp:84-85)
      camera_to_grid(poses[slot], org, f.rot, f.trans);
      vxm::set_ray_consts(f, c->cfg.grid.vox_size);
      if (depth_dev_base) f.depth = depth_dev_base + frame_elems * slot;
      f.cur = c->cur[s] ^ static_cast<uint32_t>(range & 1);  // each chained range flips the buffers
      f.occ_s = c->occ + c->n * slot;
      f.key_s = c->key + c->n * slot;
      int32_t off[3];
      const bool moved = shift_decision(c->cfg.grid, org, poses[slot].translation, off);
      for (int a = 0; a < 3; ++a) {
        f.off[a] = off[a];
        c->last_off[3 * slot + a] = off[a];
        c->origin_after[3 * slot + a] = org[a];
        P[a] += off[a];
        lo[a] = std::min(lo[a], P[a]);
        hi[a] = std::max(hi[a], P[a]);
      }
      c->last_shifted[slot] = moved ? 1 : 0;
      // epoch-tagged cells need no per-frame reset; the 8-bit epoch wraps
      // every 255 frames, when this slot's arrays are cleared once
      if (c->epoch[slot] >= vxm::kMaxEpoch) {
        c->wrapped.push_back(slot);  // cleared by run_frame on the stream that owns the slot
        c->epoch[slot] = 0;
      }
      c->epoch[slot] += 1;
      f.epoch = c->epoch[slot];
    }
    // chain box of the stream (merge_sequence_kernel): g in [min P, max P + dims)
    vxm::FrameParams& f0 = c->frames_host[s * c->F + k0];
    for (int a = 0; a < 3; ++a) {
      f0.box_lo[a] = lo[a];
      f0.box_ext[a] = hi[a] - lo[a] + c->cfg.grid.dims[a];
    }
  }
  // upload into the buffer the call before last used, on the param stream,
  // so the copy runs while the previous graph is still executing
  c->pp = (c->pp + 1) % vxm_ctx::kPP;
  const int pp = c->pp;
  if (c->sync_call) {
    // a synchronous call (the stream is idle): the copy goes on the stream
    // itself, without the cross-stream events
    VXM_CK(cudaMemcpyAsync(c->frames_pp[pp], c->frames_host, sizeof(vxm::FrameParams) * c->nslots,
                           cudaMemcpyHostToDevice, c->stream));
    VXM_CK(cudaEventRecord(c->ring_ev[c->ring_slot], c->stream));
    VXM_CK(cudaEventRecord(c->pp_ready[pp], c->stream));  // (inputs ready for desynchronised branches)
  } else {
    VXM_CK(cudaStreamWaitEvent(c->param_stream, c->pp_free[pp], 0));
    VXM_CK(cudaMemcpyAsync(c->frames_pp[pp], c->frames_host, sizeof(vxm::FrameParams) * c->nslots,
                           cudaMemcpyHostToDevice, c->param_stream));
    VXM_CK(cudaEventRecord(c->ring_ev[c->ring_slot], c->param_stream));
    VXM_CK(cudaEventRecord(c->pp_ready[pp], c->param_stream));
    VXM_CK(cudaStreamWaitEvent(c->stream, c->pp_ready[pp], 0));
  }
  c->kp.frames = c->frames_pp[pp];
}

// Clears the arrays of the wrapped slots in [s0, s0 + S) on stream st.
void clear_wrapped(vxm_ctx* c, int s0, int S, cudaStream_t st) {
  for (int slot : c->wrapped) {
    if (slot < s0 || slot >= s0 + S) continue;
    VXM_CK(cudaMemsetAsync(c->occ + c->n * slot, 0, c->n, st));
    if (c->ctr) VXM_CK(cudaMemsetAsync(c->ctr + c->n * slot, 0, c->n, st));
    if (c->rowflag) VXM_CK(cudaMemsetAsync(c->rowflag + c->rows * slot, 0, c->rows, st));
    // epoch keys are cleared with the rest; clear-format keys are all
    // Unknown after every merge already
    if (c->key_fmt == vxm::kEpochKeys) VXM_CK(cudaMemsetAsync(c->key + c->n * slot, 0, sizeof(uint32_t) * c->n, st));
  }
}

// Graph of branch b's stages (slots [s0, s1)) on its own stream.
cudaGraphExec_t capture_branch(vxm_ctx* c, int s0, int S, cudaStream_t st) {
  cudaGraph_t g = nullptr;
  VXM_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  try {
    launch_stages(c, false, true, s0, S, st, false, true);
  } catch (...) {
    cudaStreamEndCapture(st, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  VXM_CK(cudaStreamEndCapture(st, &g));
  cudaGraphExec_t exec = nullptr;
  VXM_CK(cudaGraphInstantiate(&exec, g, 0));
  VXM_CK(cudaGraphDestroy(g));
  return exec;
}

bool stage_events_wanted(const vxm_ctx* c) {
  if (c->flags & VXM_FLAG_STAGE_EVENTS) return true;
  for (void* e : c->user_stage_ev)
    if (e) return true;
  return false;
}

void run_frame(vxm_ctx* c, bool cloud, bool direct = false) {
  const bool timed = (c->flags & VXM_FLAG_STAGE_TIMING) != 0;
  const int B = graph_branches(c);
  const bool graphs = !(timed || direct || (c->flags & VXM_FLAG_NO_GRAPH));
  bool desync_call = false;
  cudaEvent_t user_input = c->user_input;  // (one call)
  c->user_input = nullptr;
  cudaEvent_t snap_ev = nullptr;
  if (c->snap_wait_pending) {
    // a snapshot's D2H reads the current local buffers: this call's kernels
    // (its merge writes the other buffer, the next call's this one) start
    // after it; the copy itself waits only for the calls issued before it
    c->snap_wait_pending = false;
    snap_ev = c->snap_copied;
    VXM_CK(cudaStreamWaitEvent(c->stream, snap_ev, 0));
  }
  if (graphs && !cloud && (c->F == 1 || c->S >= B) && B > 1 && !stage_events_wanted(c) &&
      !(c->flags & VXM_FLAG_NO_DESYNC)) {
    // Desynchronised batch: branch b's graph (its streams' stages) runs on
    // its own stream and waits only for this call's FrameParams and inputs,
    // not for the other branches of the previous call, so the branches drift
    // apart and the ALU-bound trace of one overlaps the memory-bound stages
    // of another across calls; the context stream joins them (measured:
    // 64 streams 0.238 -> 0.220 ms per call back to back).
    const int gi = c->pop_compact ? 2 : 0;
    const int pp = c->pp;
    desync_call = true;
    VXM_CK(cudaEventRecord(c->ev[0], c->stream));
    for (int b = 0; b < B; ++b) {
      if (!c->dside[b]) {
        VXM_CK(cudaStreamCreateWithFlags(&c->dside[b], cudaStreamNonBlocking));
        VXM_CK(cudaEventCreateWithFlags(&c->ddone[b], cudaEventDisableTiming));
        VXM_CK(cudaEventCreate(&c->bstart[b]));
      }
      const int s0 = c->S * b / B * c->F, s1 = c->S * (b + 1) / B * c->F;  // whole streams
      cudaStream_t bs = c->dside[b];
      if (c->tail_pending) VXM_CK(cudaStreamWaitEvent(bs, c->tail_ev, 0));
      VXM_CK(cudaStreamWaitEvent(bs, c->pp_ready[pp], 0));
      if (c->input_ready) VXM_CK(cudaStreamWaitEvent(bs, c->input_ready, 0));
      if (user_input) VXM_CK(cudaStreamWaitEvent(bs, user_input, 0));
      if (snap_ev) VXM_CK(cudaStreamWaitEvent(bs, snap_ev, 0));
      clear_wrapped(c, s0, s1 - s0, bs);
      cudaGraphExec_t& g = c->bgraph[gi][pp][b];
      if (!g) g = capture_branch(c, s0, s1 - s0, bs);
      // the branch may start before ev[0] (recorded behind the previous
      // call's joins) fires: the frame time runs from the earliest branch start
#ifndef VXM_NO_BSTART
      VXM_CK(cudaEventRecord(c->bstart[b], bs));
#endif
      VXM_CK(cudaGraphLaunch(g, bs));
      VXM_CK(cudaEventRecord(c->ddone[b], bs));
      VXM_CK(cudaStreamWaitEvent(c->stream, c->ddone[b], 0));
    }
    c->last_marks = false;
  } else if (graphs && !cloud && merge_ranges(c) > 1 && !stage_events_wanted(c) &&
             !(c->flags & VXM_FLAG_NO_DESYNC)) {
    // One stream, F >= 32 frames per call, desynchronised the same way: branch
    // b populates and traces its frame range on its own stream as soon as
    // this call's inputs are there, then merges the range as a chain after
    // the previous range's merge (range 0 after the previous call's last
    // range), so the next call's populate and trace overlap this call's chain
    // merges. Direct launches (ten per call).
    const int pp = c->pp;
    desync_call = true;
    VXM_CK(cudaEventRecord(c->ev[0], c->stream));
    for (int b = 0; b < B; ++b) {
      if (!c->dside[b]) {
        VXM_CK(cudaStreamCreateWithFlags(&c->dside[b], cudaStreamNonBlocking));
        VXM_CK(cudaEventCreateWithFlags(&c->ddone[b], cudaEventDisableTiming));
        VXM_CK(cudaEventCreate(&c->bstart[b]));
      }
      if (!c->chain[b]) VXM_CK(cudaEventCreateWithFlags(&c->chain[b], cudaEventDisableTiming));
    }
    for (int b = 0; b < B; ++b) {
      const int s0 = c->nslots * b / B, s1 = c->nslots * (b + 1) / B;
      cudaStream_t bs = c->dside[b];
      if (c->tail_pending) VXM_CK(cudaStreamWaitEvent(bs, c->tail_ev, 0));
      VXM_CK(cudaStreamWaitEvent(bs, c->pp_ready[pp], 0));
      if (c->input_ready) VXM_CK(cudaStreamWaitEvent(bs, c->input_ready, 0));
      if (user_input) VXM_CK(cudaStreamWaitEvent(bs, user_input, 0));
      if (snap_ev) VXM_CK(cudaStreamWaitEvent(bs, snap_ev, 0));
      clear_wrapped(c, s0, s1 - s0, bs);
      VXM_CK(cudaEventRecord(c->bstart[b], bs));
      launch_stages(c, false, false, s0, s1 - s0, bs, false, false);
      VXM_CK(cudaStreamWaitEvent(bs, c->chain[b == 0 ? B - 1 : b - 1], 0));
      vxm::KParams kp = c->kp;
      kp.frames += s0;
      kp.counters += s0;
      kp.counters_out += s0;
      kp.occ += c->n * s0;
      kp.key += c->n * s0;
      if (!launch_merge_chain(c, kp, s1 - s0, 1, bs)) launch_publish(kp, s1 - s0, bs);
      VXM_CK(cudaEventRecord(c->chain[b], bs));
      VXM_CK(cudaEventRecord(c->ddone[b], bs));
      VXM_CK(cudaStreamWaitEvent(c->stream, c->ddone[b], 0));
    }
    c->last_marks = false;
  } else if (!graphs) {
    if (user_input) VXM_CK(cudaStreamWaitEvent(c->stream, user_input, 0));
    clear_wrapped(c, 0, c->nslots, c->stream);
    VXM_CK(cudaEventRecord(c->ev[0], c->stream));
    launch_frame(c, cloud, false);
    c->last_marks = true;
  } else {
    const int gi = cloud ? 1 : (c->pop_compact ? 2 : 0);
    const int pp = c->pp;
    cudaGraphExec_t& g = c->graph_exec[gi][pp];
    const bool marks = stage_events_wanted(c);
    if (g && c->graph_marks[gi][pp] != marks) {  // recapture with / without the event nodes
      VXM_CK(cudaGraphExecDestroy(g));
      VXM_CK(cudaGraphDestroy(c->graph_tmpl[gi][pp]));
      g = nullptr;
      c->graph_tmpl[gi][pp] = nullptr;
      for (auto& n : c->stage_nodes[gi][pp]) n = nullptr;
    }
    if (!g) {
      g = capture(c, cloud, gi, pp, marks);
      c->stage_clean[gi][pp] = false;
    }
    if (!c->stage_clean[gi][pp]) {
      apply_stage_events(c, g, gi, pp);
      c->stage_clean[gi][pp] = true;
    }
    if (user_input) VXM_CK(cudaStreamWaitEvent(c->stream, user_input, 0));
    clear_wrapped(c, 0, c->nslots, c->stream);
    VXM_CK(cudaEventRecord(c->ev[0], c->stream));
    VXM_CK(cudaGraphLaunch(g, c->stream));
    c->last_marks = marks;
  }
  VXM_CK(cudaEventRecord(c->ev[5], c->stream));
  VXM_CK(cudaEventRecord(c->pp_free[c->pp], c->stream));  // its FrameParams may be overwritten
#ifndef VXM_NO_BSTART
  c->desync_started = desync_call ? B : 0;
#endif
  if (desync_call) {
    c->tail_pending = false;
  } else {
    // a later desynchronised call's branches start only after this call
    if (!c->tail_ev) VXM_CK(cudaEventCreateWithFlags(&c->tail_ev, cudaEventDisableTiming));
    VXM_CK(cudaEventRecord(c->tail_ev, c->stream));
    c->tail_pending = true;
  }
  const uint32_t flips = static_cast<uint32_t>(merge_ranges(c) & 1);  // K4 wrote the other buffer
  for (int s = 0; s < c->S; ++s) c->cur[s] ^= flips;
  c->pending = true;
}

void collect_stats(vxm_ctx* c, vxm_stats* out) {
  VXM_CK(cudaStreamSynchronize(c->stream));
  if (c->pending) {
    VXM_CK(cudaEventElapsedTime(&c->last_ms, c->ev[0], c->ev[5]));
    for (int b = 0; b < c->desync_started; ++b) {
      float ms = 0.f;
      VXM_CK(cudaEventElapsedTime(&ms, c->bstart[b], c->ev[5]));
      c->last_ms = std::max(c->last_ms, ms);
    }
    c->pending = false;
  }
  // K1 variant for the next frames: compact the valid pixels when fewer than
  // half of the last frames' pixels were valid (depth path only)
  {
    unsigned long long pts = 0;
    for (int s = 0; s < c->nslots; ++s) pts += c->counters_host[s].points_total;
    const double npix = static_cast<double>(c->kp.W) * c->kp.H * c->nslots;
    c->pop_compact = static_cast<double>(pts) < 0.5 * npix;
  }
  if (!out) return;
  for (int s = 0; s < c->nslots; ++s) {
    const vxm::CountersHead& k = c->counters_host[s];
    vxm_stats& o = out[s];
    std::memset(&o, 0, sizeof(o));
    o.points_total = k.points_total;
    o.points_outside = k.points_outside;
    o.rays_traced = k.rays_traced;
    o.voxels_freed = k.voxels_freed;
    o.voxels_marked_unknown_traced = k.voxels_traced;
    o.voxels_skipped_out_of_bounds = k.voxels_skipped;
    o.occupied_count = k.occupied;
    o.freed_count = k.freed;
    o.shifted = c->last_shifted[s];
    for (int a = 0; a < 3; ++a) {
      o.shift_offset[a] = c->last_off[3 * s + a];
      o.origin[a] = c->origin_after[3 * s + a];
    }
    // stage device times from the kernels' %globaltimer stamps (populate
    // includes the dilation; a stage whose stamps are missing reads 0)
    auto span_us = [](unsigned long long a, unsigned long long b) {
      return a && b && b > a ? static_cast<double>(b - a) * 1e-3 : 0.0;
    };
    o.populate_us = span_us(k.t_pop, k.t_trace);
    o.trace_us = span_us(k.t_trace, k.t_merge);
    o.merge_us = span_us(k.t_merge, k.t_end);
    o.shift_us = 0.0;  // fused into the merge kernel
  }
}

// waits for a pending asynchronous snapshot's copy and file (keeps its status
// for vxm_snapshot_wait)
void snapshot_quiesce(vxm_ctx* c) {
  if (c->snap_thread.joinable()) c->snap_thread.join();
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void destroy_ctx(vxm_ctx* c) {
  if (!c) return;
  if (c->device >= 0) cudaSetDevice(c->device);
  if (c->snap_thread.joinable()) c->snap_thread.join();
  if (c->snap_stream) {
    cudaStreamSynchronize(c->snap_stream);
    cudaStreamDestroy(c->snap_stream);
  }
  if (c->snap_start) cudaEventDestroy(c->snap_start);
  if (c->snap_copied) cudaEventDestroy(c->snap_copied);
  if (c->snap_host) cudaFreeHost(c->snap_host);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& gg : c->graph_exec)
    for (auto& g : gg)
      if (g) cudaGraphExecDestroy(g);
  for (auto& g3 : c->bgraph)
    for (auto& g2 : g3)
      for (auto& g : g2)
        if (g) cudaGraphExecDestroy(g);
  for (auto& gg : c->graph_tmpl)
    for (auto& g : gg)
      if (g) cudaGraphDestroy(g);
  if (c->param_stream) cudaStreamSynchronize(c->param_stream);
  if (c->tail_ev) cudaEventDestroy(c->tail_ev);
  for (int b = 0; b < vxm_ctx::kPP; ++b) {
    if (c->pp_ready[b]) cudaEventDestroy(c->pp_ready[b]);
    if (c->pp_free[b]) cudaEventDestroy(c->pp_free[b]);
    cudaFree(c->frames_pp[b]);
  }
  if (c->param_stream) cudaStreamDestroy(c->param_stream);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ring_ev)
    if (e) cudaEventDestroy(e);
  cudaFree(c->occ);
  cudaFree(c->ctr);
  cudaFree(c->rowflag);
  cudaFree(c->key);
  cudaFree(c->qtab);
  cudaFree(c->dbits);
  cudaFree(c->dtmp);
  cudaFree(c->loc[0]);
  cudaFree(c->loc[1]);
  cudaFree(c->counters);
  cudaFree(c->depth_dev);
  cudaFree(c->cloud_dev);
  cudaFreeHost(c->frames_ring);
  cudaFreeHost(c->counters_host);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    for (int b = 0; b < 2; ++b) {
      cudaFree(c->stage[b]);
      cudaEventDestroy(c->ev_copied[b]);
      cudaEventDestroy(c->ev_consumed[b]);
    }
    cudaStreamDestroy(c->copy_stream);
  }
  for (int b = 0; b < vxm_ctx::kBranches; ++b) {
    if (c->side[b]) cudaStreamDestroy(c->side[b]);
    if (c->fork[b]) cudaEventDestroy(c->fork[b]);
    if (c->join[b]) cudaEventDestroy(c->join[b]);
    if (c->chain[b]) cudaEventDestroy(c->chain[b]);
    if (c->dside[b]) {
      cudaStreamSynchronize(c->dside[b]);
      cudaStreamDestroy(c->dside[b]);
    }
    if (c->ddone[b]) cudaEventDestroy(c->ddone[b]);
    if (c->bstart[b]) cudaEventDestroy(c->bstart[b]);
  }
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// Drop the unused helper warning: pinned-ness is decided by the driver.
[[maybe_unused]] static bool (*const kIsPinned)(const void*) = is_pinned;

// PipelineConfig::validate (pipeline.cpp:33-42) + the GPU's own limits.
void validate_config(const vxm_config& cfg) {
  camera_validate(cfg.camera);
  if (cfg.vox_inf < 0) throw InvalidArg{"IntegratorConfig: vox_inf must be non-negative"};
  const vxm_grid_spec& g = cfg.grid;
  if (g.dims[0] < 1 || g.dims[1] < 1 || g.dims[2] < 1)
    throw InvalidArg{"PipelineConfig: empty grid"};
  if (!(cfg.depth > 0.0) || cfg.depth > cfg.camera.max_depth)
    throw InvalidArg{"PipelineConfig: depth must lie in (0, camera.max_depth]"};
  if (!(g.vox_size > 0.0)) throw InvalidArg{"vox_size must be positive"};
  // 32-bit cell indices (modular arithmetic, 0xFFFFFFFF is the tracer's
  // "no cell"): up to 2^32 - 2 cells (a 4 GB grid), x-rows counted in int
  if (static_cast<long long>(g.dims[0]) * g.dims[1] * g.dims[2] > 0xFFFFFFFELL ||
      static_cast<long long>(g.dims[1]) * g.dims[2] >= (1LL << 31))
    throw InvalidArg{"grids of more than 2^32 - 2 cells (or 2^31 x-rows) are not supported"};
}

}  // namespace

extern "C" {

const char* vxm_last_error(void) { return g_err.c_str(); }

const char* vxm_build_info(void) {
  return "cuda-sm100a voxmap kernels (fp64 IEEE, -fmad=false), ABI " "1";
}

int vxm_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int n = 0;
  for (int d = 0; d < count; ++d) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10) ++n;
  }
  return n;
}

int vxm_grid_spec_create(double sx, double sy, double sz, double vs, const double origin[3],
                         vxm_grid_spec* out) {
  const double zero[3] = {0, 0, 0};
  return guarded([&] { spec_create(sx, sy, sz, vs, origin ? origin : zero, out); });
}

int vxm_grid_spec_create_centered(double sx, double sy, double sz, double vs,
                                  const double center[3], vxm_grid_spec* out) {
  return guarded([&] {
    const double zero[3] = {0, 0, 0};
    spec_create(sx, sy, sz, vs, zero, out);
    for (int a = 0; a < 3; ++a) out->origin[a] = center[a] - half_extent(*out, a);
    if (!all_finite(out->origin, 3)) throw InvalidArg{"grid center must be finite"};
  });
}

int vxm_bundle_dimensions(const vxm_camera* cam, double depth, double vs, int32_t out[3]) {
  return guarded([&] { bundle_dims(*cam, depth, vs, out); });
}

int vxm_create(const vxm_config* cfg, int32_t n_streams, int32_t device, uint32_t flags,
               vxm_ctx** out) {
  return vxm_create_multi(cfg, n_streams, 1, device, flags, out);
}

int vxm_create_multi(const vxm_config* cfg, int32_t n_streams, int32_t frames_per_call,
                     int32_t device, uint32_t flags, vxm_ctx** out) {
  if (out) *out = nullptr;
  vxm_ctx* c = nullptr;
  const int rc = guarded([&] {
    if (!cfg || !out) throw InvalidArg{"null argument"};
    if (n_streams < 1) throw InvalidArg{"n_streams must be >= 1"};
    if (frames_per_call < 1 || frames_per_call > vxm::kMaxFramesPerCall)
      throw InvalidArg{"frames_per_call must lie in [1, " + std::to_string(vxm::kMaxFramesPerCall) + "]"};
    validate_config(*cfg);
    check_device(device);
    VXM_CK(cudaSetDevice(device));
    c = new vxm_ctx();
    c->device = device;
    c->cfg = *cfg;
    c->S = n_streams;
    c->F = frames_per_call;
    c->nslots = n_streams * frames_per_call;
    c->flags = flags;
    c->nsm = sm_count(device);
    const vxm_grid_spec& g = cfg->grid;
    c->n = static_cast<long long>(g.dims[0]) * g.dims[1] * g.dims[2];
    c->rows = static_cast<long long>(g.dims[1]) * g.dims[2];
    bundle_dims(cfg->camera, cfg->depth, g.vox_size, c->bundle);
    const long long rays = static_cast<long long>(c->bundle[1]) * c->bundle[2];
    if (rays > vxm::kMaxClearRays)
      throw InvalidArg{"ray bundle exceeds " + std::to_string(vxm::kMaxClearRays) + " rays"};
    // epoch-tagged keys whenever the bundle fits their 17-bit ray field
    c->key_fmt = rays <= vxm::kMaxEpochRays && !(flags & VXM_FLAG_CLEAR_KEYS) ? vxm::kEpochKeys : vxm::kClearKeys;

    VXM_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (auto& e : c->ev) VXM_CK(cudaEventCreate(&e));
    const size_t S = static_cast<size_t>(c->nslots);  // measurement-grid slots
    const size_t NS = static_cast<size_t>(n_streams);  // local grids
    const size_t npix = static_cast<size_t>(cfg->camera.width) * cfg->camera.height;
    // 64 bytes of slack after each array: the TMA-staged K4 reads windows
    // widened to 16-byte boundaries
    VXM_CK(cudaMalloc(&c->occ, c->n * S + 64));
    VXM_CK(cudaMemsetAsync(c->occ, 0, c->n * S, c->stream));
    VXM_CK(cudaMalloc(&c->key, sizeof(uint32_t) * c->n * S + 64));
    VXM_CK(cudaMemsetAsync(c->key, 0, sizeof(uint32_t) * c->n * S, c->stream));
    if (cfg->vox_inf > 0) {
      VXM_CK(cudaMalloc(&c->ctr, c->n * S));
      VXM_CK(cudaMemsetAsync(c->ctr, 0, c->n * S, c->stream));
      VXM_CK(cudaMalloc(&c->rowflag, c->rows * S));
      VXM_CK(cudaMemsetAsync(c->rowflag, 0, c->rows * S, c->stream));
    }
    for (int b = 0; b < 2; ++b) {
      VXM_CK(cudaMalloc(&c->loc[b], c->n * NS + 64));
      VXM_CK(cudaMemsetAsync(c->loc[b], 0, c->n * NS, c->stream));
    }
    VXM_CK(cudaMalloc(&c->counters, sizeof(vxm::Counters) * S));
    VXM_CK(cudaMemsetAsync(c->counters, 0, sizeof(vxm::Counters) * S, c->stream));  // then cleared by K4
    for (int b = 0; b < vxm_ctx::kPP; ++b) {
      VXM_CK(cudaMalloc(&c->frames_pp[b], sizeof(vxm::FrameParams) * S));
      VXM_CK(cudaEventCreateWithFlags(&c->pp_ready[b], cudaEventDisableTiming));
      VXM_CK(cudaEventCreateWithFlags(&c->pp_free[b], cudaEventDisableTiming));
    }
    VXM_CK(cudaStreamCreateWithFlags(&c->param_stream, cudaStreamNonBlocking));
    VXM_CK(cudaMalloc(&c->depth_dev, sizeof(float) * npix * S));
    VXM_CK(cudaMallocHost(&c->frames_ring, sizeof(vxm::FrameParams) * S * vxm_ctx::kRing));
    std::memset(c->frames_ring, 0, sizeof(vxm::FrameParams) * S * vxm_ctx::kRing);
    for (auto& e : c->ring_ev) VXM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->frames_host = c->frames_ring;
    VXM_CK(cudaHostAlloc(&c->counters_host, sizeof(vxm::CountersHead) * S, cudaHostAllocMapped));
    std::memset(c->counters_host, 0, sizeof(vxm::CountersHead) * S);

    c->epoch.assign(S, 0);
    c->cur.assign(NS, 0);
    c->origin.resize(3 * NS);
    c->last_off.assign(3 * S, 0);
    c->last_shifted.assign(S, 0);
    c->origin_after.resize(3 * S);
    for (size_t s = 0; s < NS; ++s)
      for (int a = 0; a < 3; ++a) c->origin[3 * s + a] = g.origin[a];
    for (size_t s = 0; s < S; ++s)
      for (int a = 0; a < 3; ++a) c->origin_after[3 * s + a] = g.origin[a];

    vxm::KParams& kp = c->kp;
    kp.dx = g.dims[0];
    kp.dy = g.dims[1];
    kp.dz = g.dims[2];
    kp.n = c->n;
    kp.vs = g.vox_size;
    kp.W = cfg->camera.width;
    kp.H = cfg->camera.height;
    // CameraModel::focal_x/y (geometry.hpp:67-68) and the principal point
    // (geometry.cpp:50-51), computed once on the host with glibc tan; the
    // per-column / per-row factors ((u + 0.5) - cx) / fx of back_project_rows
    // (geometry.cpp:55-56) are tabulated with the same IEEE operations.
    {
      const double fx = (cfg->camera.width / 2.0) / std::tan(cfg->camera.fov_x / 2.0);
      const double fy = (cfg->camera.height / 2.0) / std::tan(cfg->camera.fov_y / 2.0);
      const double cx = cfg->camera.width / 2.0;
      const double cy = cfg->camera.height / 2.0;
      std::vector<double> q(static_cast<size_t>(kp.W) + kp.H);
      for (int u = 0; u < kp.W; ++u) q[u] = ((u + 0.5) - cx) / fx;
      for (int v = 0; v < kp.H; ++v) q[kp.W + v] = ((v + 0.5) - cy) / fy;
      VXM_CK(cudaMalloc(&c->qtab, sizeof(double) * q.size()));
      VXM_CK(cudaMemcpy(c->qtab, q.data(), sizeof(double) * q.size(), cudaMemcpyHostToDevice));
      kp.qx = c->qtab;
      kp.qy = c->qtab + kp.W;
    }
    kp.inv_vs = 1.0 / g.vox_size;
    kp.ray_vs = g.vox_size;
    kp.max_depth = cfg->camera.max_depth;
    kp.max_depth_f = vxm::max_float_at_most(cfg->camera.max_depth);
    kp.vox_inf = cfg->vox_inf;
    kp.vd = c->bundle[0];
    kp.vw = c->bundle[1];
    kp.vh = c->bundle[2];
    kp.tiles_x = (kp.vw + 7) / 8;
    kp.tiles_y = (kp.vh + 3) / 4;
    for (const void* fn : {reinterpret_cast<const void*>(vxm::merge_epoch_tma_kernel),
                           reinterpret_cast<const void*>(vxm::merge_shift_count_tma_kernel<true>)})
      VXM_CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(2 * vxm::merge_tma_smem_bytes(vxm::kMergeStageCells))));
    for (const void* fn : {reinterpret_cast<const void*>(vxm::populate_depth_tma_kernel<true, false>),
                           reinterpret_cast<const void*>(vxm::populate_depth_tma_kernel<false, false>),
                           reinterpret_cast<const void*>(vxm::populate_depth_tma_kernel<true, true>),
                           reinterpret_cast<const void*>(vxm::populate_depth_tma_kernel<false, true>)})
      VXM_CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>((sizeof(float4) + 4 * sizeof(uint16_t)) * kPopulateThreads *
                                                   vxm::kPopMaxIters)));
    kp.occ = c->occ;
    kp.ctr = c->ctr;
    kp.rowflag = c->rowflag;
    kp.key = c->key;
    kp.key_fmt = c->key_fmt;
    kp.loc0 = c->loc[0];
    kp.loc1 = c->loc[1];
    kp.counters = c->counters;
    VXM_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&kp.counters_out), c->counters_host, 0));

    kp.frames = c->frames_pp[0];
    if (cfg->vox_inf > 0) {
      if (vxm::dilate_generic(cfg->vox_inf, kp.dx)) {
        // radii / rows beyond the tile kernels: the generic line passes
        VXM_CK(cudaMalloc(&c->dtmp, 2 * static_cast<size_t>(c->n) * S));
        kp.dtmp = c->dtmp;
      } else {
        const size_t words = static_cast<size_t>(vxm::dilate_row_words(kp.dx)) * kp.dy * kp.dz * S;
        VXM_CK(cudaMalloc(&c->dbits, sizeof(uint32_t) * words));
        kp.dbits = c->dbits;
        VXM_CK(vxm::dilate_set_smem(static_cast<int>(
            vxm::dilate_smem_bytes(cfg->vox_inf, kp.dx, vxm::dilate_fused(cfg->vox_inf, kp.dx)))));
      }
    }
    VXM_CK(cudaStreamSynchronize(c->stream));
  });
  if (rc != VXM_OK) {
    destroy_ctx(c);
    return rc;
  }
  *out = c;
  return VXM_OK;
}

int vxm_destroy(vxm_ctx* ctx) {
  destroy_ctx(ctx);
  return VXM_OK;
}

int vxm_num_streams(const vxm_ctx* ctx) { return ctx ? ctx->S : 0; }

int vxm_frames_per_call(const vxm_ctx* ctx) { return ctx ? ctx->F : 0; }

int vxm_graph_branches(const vxm_ctx* ctx) { return ctx ? graph_branches(ctx) : 0; }

void* vxm_cuda_stream(vxm_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int vxm_last_frame_ms(vxm_ctx* ctx, float* ms) {
  return guarded([&] {
    collect_stats(ctx, nullptr);
    *ms = ctx->last_ms;
  });
}

int vxm_integrate_depth(vxm_ctx* ctx, const float* depth, const vxm_pose* t_wc, vxm_stats* stats) {
  return guarded([&] {
    if (!ctx || !depth || !t_wc) throw InvalidArg{"null argument"};
    VXM_CK(cudaSetDevice(ctx->device));
    const size_t frame = static_cast<size_t>(ctx->kp.W) * ctx->kp.H;
    next_slot(ctx);
    // pinned host buffers go straight to the copy engine; pageable ones are
    // staged by the driver
    VXM_CK(cudaMemcpyAsync(ctx->depth_dev, depth, sizeof(float) * frame * ctx->nslots,
                           cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync_call = true;
    try {
      prepare_frames(ctx, t_wc, ctx->depth_dev, frame);
    } catch (...) {
      ctx->sync_call = false;
      throw;
    }
    ctx->sync_call = false;
    run_frame(ctx, false);
    collect_stats(ctx, stats);
  });
}

int vxm_integrate_depth_frames(vxm_ctx* ctx, const float* depth, const vxm_pose* t_wc, int32_t n_frames,
                               vxm_stats* stats) {
  return guarded([&] {
    if (!ctx || !depth || !t_wc) throw InvalidArg{"null argument"};
    if (ctx->S != 1) throw InvalidArg{"vxm_integrate_depth_frames needs a single-stream context"};
    if (n_frames < 1 || n_frames > ctx->F) throw InvalidArg{"n_frames must lie in [1, frames_per_call]"};
    VXM_CK(cudaSetDevice(ctx->device));
    const size_t frame = static_cast<size_t>(ctx->kp.W) * ctx->kp.H;
    const int F = ctx->F;
    // a shorter call runs the first n_frames slots with direct launches (the
    // captured graph has the full shape); slots keep their own epochs
    ctx->F = ctx->nslots = n_frames;
    try {
      next_slot(ctx);
      // the depth copy goes first on the context stream and the call is
      // synchronous, so FrameParams (and pp_ready, which the desynchronised
      // chained-range branches wait on) are recorded after the copy
      VXM_CK(cudaMemcpyAsync(ctx->depth_dev, depth, sizeof(float) * frame * n_frames,
                             cudaMemcpyHostToDevice, ctx->stream));
      ctx->sync_call = true;
      prepare_frames(ctx, t_wc, ctx->depth_dev, frame);
      ctx->sync_call = false;
      run_frame(ctx, false, n_frames != F);
      collect_stats(ctx, stats);
    } catch (...) {
      ctx->sync_call = false;
      ctx->F = ctx->nslots = F;
      throw;
    }
    ctx->F = ctx->nslots = F;
  });
}

int vxm_integrate_depth_device(vxm_ctx* ctx, const float* depth_dev, const vxm_pose* t_wc) {
  return guarded([&] {
    if (!ctx || !depth_dev || !t_wc) throw InvalidArg{"null argument"};
    VXM_CK(cudaSetDevice(ctx->device));
    const size_t frame = static_cast<size_t>(ctx->kp.W) * ctx->kp.H;
    next_slot(ctx);
    prepare_frames(ctx, t_wc, depth_dev, frame);
    run_frame(ctx, false);
  });
}

// Host-buffer frames, asynchronous and double buffered: the H2D copy of this
// call runs on the context's copy stream into one of two staging buffers
// while the compute stream may still be busy with the previous frame.
int vxm_integrate_depth_async(vxm_ctx* ctx, const float* depth, const vxm_pose* t_wc) {
  return guarded([&] {
    if (!ctx || !depth || !t_wc) throw InvalidArg{"null argument"};
    VXM_CK(cudaSetDevice(ctx->device));
    const size_t frame = static_cast<size_t>(ctx->kp.W) * ctx->kp.H;
    const size_t bytes = sizeof(float) * frame * ctx->nslots;
    if (!ctx->copy_stream) {
      VXM_CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        VXM_CK(cudaMalloc(&ctx->stage[b], bytes));
        VXM_CK(cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming));
        VXM_CK(cudaEventCreateWithFlags(&ctx->ev_consumed[b], cudaEventDisableTiming));
        VXM_CK(cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
      }
    }
    const int b = ctx->stage_slot;
    ctx->stage_slot ^= 1;
    VXM_CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_consumed[b], 0));  // K1 done with it
    VXM_CK(cudaMemcpyAsync(ctx->stage[b], depth, bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
    VXM_CK(cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
    next_slot(ctx);
    prepare_frames(ctx, t_wc, ctx->stage[b], frame);
    VXM_CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0));
    ctx->input_ready = ctx->ev_copied[b];  // (desynchronised branches wait on it themselves)
    run_frame(ctx, false);
    ctx->input_ready = nullptr;
    VXM_CK(cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
  });
}

int vxm_set_input_event(vxm_ctx* ctx, void* cuda_event) {
  return guarded([&] {
    if (!ctx) throw InvalidArg{"null context"};
    ctx->user_input = static_cast<cudaEvent_t>(cuda_event);
  });
}

int vxm_set_stage_events(vxm_ctx* ctx, void* const events[4]) {
  return guarded([&] {
    if (!ctx) throw InvalidArg{"null context"};
    for (int i = 0; i < 4; ++i) ctx->user_stage_ev[i] = events ? events[i] : nullptr;
    for (auto& dd : ctx->stage_clean)
      for (bool& d : dd) d = false;
  });
}

int vxm_wait_stats(vxm_ctx* ctx, vxm_stats* stats) {
  return guarded([&] {
    VXM_CK(cudaSetDevice(ctx->device));
    collect_stats(ctx, stats);
  });
}

int vxm_integrate_cloud(vxm_ctx* ctx, const double* xs, const double* ys, const double* zs,
                        size_t n, const vxm_pose* t_wc, vxm_stats* stats) {
  return guarded([&] {
    if (!ctx || !t_wc) throw InvalidArg{"null argument"};
    if (ctx->nslots != 1) throw InvalidArg{"vxm_integrate_cloud needs a single-stream, single-frame context"};
    if (n > 0 && (!xs || !ys || !zs)) throw InvalidArg{"null cloud arrays"};
    VXM_CK(cudaSetDevice(ctx->device));
    if (n > ctx->cloud_cap) {
      cudaFree(ctx->cloud_dev);
      ctx->cloud_dev = nullptr;
      ctx->cloud_cap = 0;
      VXM_CK(cudaMalloc(&ctx->cloud_dev, sizeof(double) * 3 * n));
      ctx->cloud_cap = n;
    }
    next_slot(ctx);
    vxm::FrameParams& f = ctx->frames_host[0];
    f.xs = ctx->cloud_dev;
    f.ys = ctx->cloud_dev + ctx->cloud_cap;
    f.zs = ctx->cloud_dev + 2 * ctx->cloud_cap;
    f.n_points = static_cast<long long>(n);
    prepare_frames(ctx, t_wc, nullptr, 0);
    if (n) {
      VXM_CK(cudaMemcpyAsync(const_cast<double*>(f.xs), xs, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
      VXM_CK(cudaMemcpyAsync(const_cast<double*>(f.ys), ys, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
      VXM_CK(cudaMemcpyAsync(const_cast<double*>(f.zs), zs, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    }
    run_frame(ctx, true);
    collect_stats(ctx, stats);
  });
}

int vxm_download_local(vxm_ctx* ctx, int32_t s, uint8_t* cells, double origin[3]) {
  return guarded([&] {
    if (!ctx || s < 0 || s >= ctx->S) throw InvalidArg{"stream index out of range"};
    VXM_CK(cudaSetDevice(ctx->device));
    collect_stats(ctx, nullptr);
    if (cells)
      VXM_CK(cudaMemcpy(cells, ctx->loc[ctx->cur[s]] + ctx->n * s, ctx->n, cudaMemcpyDeviceToHost));
    if (origin)
      for (int a = 0; a < 3; ++a) origin[a] = ctx->origin[3 * s + a];
  });
}

int vxm_upload_local(vxm_ctx* ctx, int32_t s, const uint8_t* cells, const double origin[3]) {
  return guarded([&] {
    if (!ctx || s < 0 || s >= ctx->S) throw InvalidArg{"stream index out of range"};
    snapshot_quiesce(ctx);  // a pending snapshot copy reads the buffer this overwrites
    if (origin && !all_finite(origin, 3)) throw InvalidArg{"grid origin must be finite"};
    VXM_CK(cudaSetDevice(ctx->device));
    collect_stats(ctx, nullptr);
    if (cells)
      VXM_CK(cudaMemcpy(ctx->loc[ctx->cur[s]] + ctx->n * s, cells, ctx->n, cudaMemcpyHostToDevice));
    if (origin)
      for (int a = 0; a < 3; ++a) ctx->origin[3 * s + a] = origin[a];
  });
}

// ---------------------------------------------------------------------------
// VOXGRID1 snapshots (proj/include/voxmap/grid_io.hpp:10-17, grid_io.cpp:14-69)
// ---------------------------------------------------------------------------
namespace {
void write_voxgrid(const char* path, const int dims[3], double vs, const double origin[3], const uint8_t* cells) {
  FILE* f = std::fopen(path, "wb");
  if (!f) throw IoError{std::string("write_grid: cannot open ") + path};
  const std::string h = vxm_io::voxgrid_header(dims, vs, origin);
  const size_t n = static_cast<size_t>(dims[0]) * dims[1] * dims[2];
  const bool ok = std::fwrite(h.data(), 1, h.size(), f) == h.size() && std::fwrite(cells, 1, n, f) == n;
  if (std::fclose(f) != 0 || !ok) throw IoError{"write_grid: stream write failed"};
}

std::vector<char> slurp(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) throw IoError{std::string("read_grid: cannot open ") + path};
  std::vector<char> buf;
  char tmp[1 << 16];
  size_t got;
  while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  std::fclose(f);
  return buf;
}

vxm_io::VoxgridHeader read_voxgrid(const std::vector<char>& buf) {
  vxm_io::VoxgridHeader h;
  std::string err = vxm_io::parse_voxgrid_header(buf.data(), buf.size(), h);
  if (err.empty()) err = vxm_io::check_voxgrid_cells(buf.data(), buf.size(), h);
  if (!err.empty()) throw IoError{err};
  return h;
}
}  // namespace

int vxm_grid_write(const char* path, const vxm_grid_spec* spec, const uint8_t* cells) {
  return guarded([&] {
    if (!path || !spec || !cells) throw InvalidArg{"null argument"};
    write_voxgrid(path, spec->dims, spec->vox_size, spec->origin, cells);
  });
}

int vxm_grid_read(const char* path, vxm_grid_spec* spec, uint8_t* cells, size_t capacity) {
  return guarded([&] {
    if (!path || !spec) throw InvalidArg{"null argument"};
    const std::vector<char> buf = slurp(path);
    const vxm_io::VoxgridHeader h = read_voxgrid(buf);
    std::memset(spec, 0, sizeof(*spec));
    for (int a = 0; a < 3; ++a) {
      spec->dims[a] = h.dims[a];
      spec->size[a] = h.dims[a] * h.vox_size;  // grid_io.cpp: grid_size = dims * vox_size
      spec->origin[a] = h.origin[a];
    }
    spec->vox_size = h.vox_size;
    if (cells) {
      if (capacity < h.cells()) throw InvalidArg{"read_grid: cell buffer too small"};
      std::memcpy(cells, buf.data() + h.data_offset, h.cells());
    }
  });
}

int vxm_snapshot_save(vxm_ctx* ctx, int32_t s, const char* path) {
  return guarded([&] {
    if (!ctx || s < 0 || s >= ctx->S) throw InvalidArg{"stream index out of range"};
    if (!path) throw InvalidArg{"null path"};
    VXM_CK(cudaSetDevice(ctx->device));
    collect_stats(ctx, nullptr);
    std::vector<uint8_t> cells(static_cast<size_t>(ctx->n));
    VXM_CK(cudaMemcpy(cells.data(), ctx->loc[ctx->cur[s]] + ctx->n * s, ctx->n, cudaMemcpyDeviceToHost));
    write_voxgrid(path, ctx->cfg.grid.dims, ctx->cfg.grid.vox_size, &ctx->origin[3 * s], cells.data());
  });
}

namespace {
// joins the writer thread of the previous asynchronous snapshot
int snapshot_join(vxm_ctx* ctx) {
  if (ctx->snap_thread.joinable()) ctx->snap_thread.join();
  const int rc = ctx->snap_status;
  if (rc != VXM_OK) g_err = ctx->snap_error;
  ctx->snap_status = VXM_OK;
  return rc;
}
}  // namespace

int vxm_snapshot_save_async(vxm_ctx* ctx, int32_t s, const char* path) {
  if (ctx) {
    const int prev = snapshot_join(ctx);
    if (prev != VXM_OK) return prev;
  }
  return guarded([&] {
    if (!ctx || s < 0 || s >= ctx->S) throw InvalidArg{"stream index out of range"};
    if (!path) throw InvalidArg{"null path"};
    VXM_CK(cudaSetDevice(ctx->device));
    if (!ctx->snap_stream) {
      VXM_CK(cudaStreamCreateWithFlags(&ctx->snap_stream, cudaStreamNonBlocking));
      VXM_CK(cudaEventCreateWithFlags(&ctx->snap_start, cudaEventDisableTiming));
      VXM_CK(cudaEventCreateWithFlags(&ctx->snap_copied, cudaEventDisableTiming));
      VXM_CK(cudaMallocHost(&ctx->snap_host, static_cast<size_t>(ctx->n)));
    }
    // the grid as it stands after every call issued so far: the context
    // stream joins each call's branches, so an event there marks that point
    VXM_CK(cudaEventRecord(ctx->snap_start, ctx->stream));
    VXM_CK(cudaStreamWaitEvent(ctx->snap_stream, ctx->snap_start, 0));
    VXM_CK(cudaMemcpyAsync(ctx->snap_host, ctx->loc[ctx->cur[s]] + ctx->n * s, static_cast<size_t>(ctx->n),
                           cudaMemcpyDeviceToHost, ctx->snap_stream));
    VXM_CK(cudaEventRecord(ctx->snap_copied, ctx->snap_stream));
    ctx->snap_wait_pending = true;
    // header fields as of now (host state: the origin after the last call)
    int dims[3];
    double origin[3];
    for (int a = 0; a < 3; ++a) {
      dims[a] = ctx->cfg.grid.dims[a];
      origin[a] = ctx->origin[3 * s + a];
    }
    const double vs = ctx->cfg.grid.vox_size;
    const std::string file(path);
    const int device = ctx->device;
    ctx->snap_thread = std::thread([ctx, dims, origin, vs, file, device]() {
      cudaSetDevice(device);
      if (cudaEventSynchronize(ctx->snap_copied) != cudaSuccess) {
        ctx->snap_status = VXM_ECUDA;
        ctx->snap_error = "snapshot copy failed";
        return;
      }
      try {
        write_voxgrid(file.c_str(), dims, vs, origin, ctx->snap_host);
      } catch (const IoError& e) {
        ctx->snap_status = VXM_EIO;
        ctx->snap_error = e.what;
      }
    });
  });
}

int vxm_snapshot_wait(vxm_ctx* ctx) {
  if (!ctx) return fail(VXM_EINVAL, "null context");
  return snapshot_join(ctx);
}

int vxm_snapshot_load(vxm_ctx* ctx, int32_t s, const char* path) {
  return guarded([&] {
    if (!ctx || s < 0 || s >= ctx->S) throw InvalidArg{"stream index out of range"};
    if (!path) throw InvalidArg{"null path"};
    const std::vector<char> buf = slurp(path);
    const vxm_io::VoxgridHeader h = read_voxgrid(buf);
    const vxm_grid_spec& g = ctx->cfg.grid;
    if (h.dims[0] != g.dims[0] || h.dims[1] != g.dims[1] || h.dims[2] != g.dims[2] || h.vox_size != g.vox_size)
      throw InvalidArg{"snapshot grid does not match the pipeline's GridSpec"};
    VXM_CK(cudaSetDevice(ctx->device));
    snapshot_quiesce(ctx);
    collect_stats(ctx, nullptr);
    VXM_CK(cudaMemcpy(ctx->loc[ctx->cur[s]] + ctx->n * s, buf.data() + h.data_offset, ctx->n,
                      cudaMemcpyHostToDevice));
    for (int a = 0; a < 3; ++a) ctx->origin[3 * s + a] = h.origin[a];
  });
}

}  // extern "C"
