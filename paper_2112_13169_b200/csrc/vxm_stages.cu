// Stand-alone stage entry points of include/vxm.h: the free functions of the
// public API operating on HOST grids (populate_occupied, trace_bundle,
// merge_grids, shift_grid_by, depth_to_cloud) and the KernelTable adapter.
// Each call uploads, runs the same kernels as the per-frame graph on the
// current device's legacy stream, and downloads. They exist for API
// completeness and parity; the hot path is vxm_integrate_* on a context.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vxm.h"
#include "vxm_aux_kernels.cuh"
#include "vxm_kernels.cuh"

// Defined in vxm_runtime.cu: the thread-local slot vxm_last_error() reads.
void vxm_set_error(const char* msg);

namespace {

struct StageError {
  int code;
  std::string what;
};

#define VXM_SCK(call)                                                                    \
  do {                                                                                   \
    const cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                               \
      throw StageError{e_ == cudaErrorMemoryAllocation ? VXM_ENOMEM : VXM_ECUDA,         \
                       std::string(#call) + ": " + cudaGetErrorString(e_)};              \
  } while (0)

// Per-thread, per-device cache of stage scratch blocks. Every stage call runs
// on its thread's default stream and ends in a synchronous download (or a
// device synchronize), so a block released at the end of one call is idle
// and the next call on the thread reuses it: no cudaMalloc/cudaFree per call
// (the reference's stage functions allocate nothing on the device). Blocks
// are rounded up to powers of two; at most kScratchKeep bytes stay cached.
struct ScratchBlock {
  int dev;
  void* p;
  size_t bytes;
  bool used;
};
constexpr size_t kScratchKeep = size_t(1) << 31;
struct ScratchCache {
  std::vector<ScratchBlock> blocks;
  size_t kept = 0;
  ~ScratchCache() {
    for (auto& b : blocks) cudaFree(b.p);  // thread exit; fails harmlessly at process teardown
  }
  void* acquire(size_t bytes) {
    int dev = 0;
    VXM_SCK(cudaGetDevice(&dev));
    ScratchBlock* best = nullptr;
    for (auto& b : blocks)
      if (!b.used && b.dev == dev && b.bytes >= bytes && (!best || b.bytes < best->bytes)) best = &b;
    if (best) {
      best->used = true;
      return best->p;
    }
    size_t cap = 256;
    while (cap < bytes) cap <<= 1;
    void* p = nullptr;
    if (cudaMalloc(&p, cap) != cudaSuccess) {  // drop the idle blocks and retry once
      cudaGetLastError();
      trim(0);
      VXM_SCK(cudaMalloc(&p, cap));
    }
    blocks.push_back({dev, p, cap, true});
    kept += cap;
    return p;
  }
  void release(void* p) {
    for (auto& b : blocks)
      if (b.p == p) b.used = false;
    trim(kScratchKeep);
  }
  void trim(size_t keep) {
    for (size_t i = blocks.size(); i-- > 0 && kept > keep;)
      if (!blocks[i].used) {
        cudaFree(blocks[i].p);
        kept -= blocks[i].bytes;
        blocks.erase(blocks.begin() + static_cast<long>(i));
      }
  }
};
thread_local ScratchCache g_scratch;

// RAII device buffer from the scratch cache.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) {
    if (n) p = static_cast<T*>(g_scratch.acquire(sizeof(T) * n));
  }
  ~DevBuf() {
    if (p) g_scratch.release(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

void require_device() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw StageError{VXM_ENODEV, "no CUDA device visible"};
  }
}

template <typename F>
int stage_guard(F&& f) {
  try {
    require_device();
    f();
    return VXM_OK;
  } catch (const StageError& e) {
    vxm_set_error(e.what.c_str());
    return e.code;
  }
}

unsigned blocks_for(long long n, int threads, int cap = 148 * 16) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<unsigned>(b);
}

constexpr uint32_t kEpoch = 1u;

// key format of a stage call, as a context would choose it
int key_fmt_for(long long rays) { return rays <= vxm::kMaxEpochRays ? vxm::kEpochKeys : vxm::kClearKeys; }

// One-stream kernel parameters for a grid (no camera, no bundle).
vxm::KParams grid_params(const vxm_grid_spec& g) {
  vxm::KParams kp{};
  kp.dx = g.dims[0];
  kp.dy = g.dims[1];
  kp.dz = g.dims[2];
  kp.n = static_cast<long long>(g.dims[0]) * g.dims[1] * g.dims[2];
  kp.vs = g.vox_size;
  kp.inv_vs = 1.0 / g.vox_size;
  kp.ray_vs = g.vox_size;
  return kp;
}

void check_grid(const vxm_grid_spec* g) {
  if (!g) throw StageError{VXM_EINVAL, "null grid spec"};
  if (g->dims[0] < 1 || g->dims[1] < 1 || g->dims[2] < 1)
    throw StageError{VXM_EINVAL, "grid must be at least one voxel per axis"};
  if (!(g->vox_size > 0.0)) throw StageError{VXM_EINVAL, "vox_size must be positive"};
  if (static_cast<long long>(g->dims[0]) * g->dims[1] * g->dims[2] > 0xFFFFFFFELL ||
      static_cast<long long>(g->dims[1]) * g->dims[2] >= (1LL << 31))
    throw StageError{VXM_EINVAL, "grids of more than 2^32 - 2 cells (or 2^31 x-rows) are not supported"};
}

void fill_pose(vxm::FrameParams& f, const vxm_pose& t) {
  std::memcpy(f.rot, t.rotation, sizeof(f.rot));
  std::memcpy(f.trans, t.translation, sizeof(f.trans));
}

}  // namespace

extern "C" {

int vxm_populate_occupied(const vxm_grid_spec* grid, uint8_t* ms, const double* xs,
                          const double* ys, const double* zs, size_t n, const vxm_pose* t_vc,
                          int32_t vox_inf, vxm_populate_stats* st) {
  return stage_guard([&] {
    check_grid(grid);
    if (vox_inf < 0) throw StageError{VXM_EINVAL, "IntegratorConfig: vox_inf must be non-negative"};
    if (!ms || !t_vc || (n && (!xs || !ys || !zs))) throw StageError{VXM_EINVAL, "null argument"};
    vxm::KParams kp = grid_params(*grid);
    const long long N = kp.n;
    DevBuf<uint8_t> d_ms(N), d_occ(N), d_ctr(vox_inf > 0 ? N : 0);
    DevBuf<uint8_t> d_rowflag(vox_inf > 0 ? static_cast<long long>(kp.dy) * kp.dz : 0);
    DevBuf<uint32_t> d_key(N);
    DevBuf<double> d_pts(3 * n + 1);
    DevBuf<vxm::Counters> d_cnt(1);
    DevBuf<vxm::FrameParams> d_frame(1);
    vxm::FrameParams f{};
    fill_pose(f, *t_vc);
    f.xs = d_pts.p;
    f.ys = d_pts.p + n;
    f.zs = d_pts.p + 2 * n;
    f.n_points = static_cast<long long>(n);
    f.epoch = kEpoch;
    VXM_SCK(cudaMemcpy(d_frame.p, &f, sizeof(f), cudaMemcpyHostToDevice));
    if (n) {
      VXM_SCK(cudaMemcpy(d_pts.p, xs, sizeof(double) * n, cudaMemcpyHostToDevice));
      VXM_SCK(cudaMemcpy(d_pts.p + n, ys, sizeof(double) * n, cudaMemcpyHostToDevice));
      VXM_SCK(cudaMemcpy(d_pts.p + 2 * n, zs, sizeof(double) * n, cudaMemcpyHostToDevice));
    }
    VXM_SCK(cudaMemcpy(d_ms.p, ms, N, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemset(d_cnt.p, 0, sizeof(vxm::Counters)));
    if (d_ctr.p) VXM_SCK(cudaMemset(d_ctr.p, 0, N));
    if (d_rowflag.p) VXM_SCK(cudaMemset(d_rowflag.p, 0, static_cast<size_t>(kp.dy) * kp.dz));
    vxm::encode_ms_kernel<<<blocks_for(N, 256), 256>>>(d_ms.p, d_occ.p, d_key.p, N, kEpoch, vxm::kEpochKeys);
    kp.occ = d_occ.p;
    kp.key = d_key.p;
    kp.key_fmt = vxm::kEpochKeys;
    kp.ctr = d_ctr.p;
    kp.rowflag = d_rowflag.p;
    kp.vox_inf = vox_inf;
    kp.counters = d_cnt.p;
    kp.frames = d_frame.p;
    vxm::populate_cloud_kernel<false><<<dim3(blocks_for(static_cast<long long>(n), 256), 1), 256>>>(kp);
    VXM_SCK(cudaGetLastError());
    const bool generic = vox_inf > 0 && vxm::dilate_generic(vox_inf, kp.dx);
    DevBuf<uint32_t> d_bits(vox_inf > 0 && !generic
                                ? static_cast<size_t>(vxm::dilate_row_words(kp.dx)) * kp.dy * kp.dz : 0);
    DevBuf<uint8_t> d_tmp(generic ? 2 * static_cast<size_t>(N) : 0);
    if (vox_inf > 0) {
      const int r = vox_inf;
      if (!generic)
        VXM_SCK(vxm::dilate_set_smem(static_cast<int>(vxm::dilate_smem_bytes(r, kp.dx, vxm::dilate_fused(r, kp.dx)))));
      kp.dbits = d_bits.p;
      kp.dtmp = d_tmp.p;
      vxm::launch_dilate(kp, r, 1, 0, 0);
      VXM_SCK(cudaGetLastError());
    }
    vxm::decode_ms_kernel<<<blocks_for(N, 256), 256>>>(d_occ.p, d_key.p, d_ms.p, N, kEpoch, vxm::kEpochKeys, 1);
    VXM_SCK(cudaGetLastError());
    vxm::Counters cnt{};
    VXM_SCK(cudaMemcpy(&cnt, d_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost));
    VXM_SCK(cudaMemcpy(ms, d_ms.p, N, cudaMemcpyDeviceToHost));
    if (st) {
      st->points_total = cnt.points_total;
      st->points_outside = cnt.points_outside;
    }
  });
}

int vxm_trace_bundle(const vxm_grid_spec* grid, uint8_t* ms, const int32_t bundle[3],
                     const vxm_pose* t_vc, double ray_vox_size, vxm_trace_stats* st) {
  return stage_guard([&] {
    check_grid(grid);
    if (!ms || !bundle || !t_vc) throw StageError{VXM_EINVAL, "null argument"};
    // generate_rays preconditions (raytracer.cpp:37-44)
    if (bundle[0] < 1 || bundle[1] < 1 || bundle[2] < 1 || bundle[1] % 2 == 0 || bundle[2] % 2 == 0)
      throw StageError{VXM_EINVAL, "generate_rays: bundle dimensions must be positive and odd"};
    if (!(ray_vox_size > 0.0)) throw StageError{VXM_EINVAL, "generate_rays: vox_size must be positive"};
    const long long rays = static_cast<long long>(bundle[1]) * bundle[2];
    if (rays > vxm::kMaxClearRays) throw StageError{VXM_EINVAL, "ray bundle exceeds 2^31 - 3 rays"};
    const int fmt = key_fmt_for(rays);
    // validate_ray (raytracer.cpp:23-33) for every ray, before any write.
    const double vs = ray_vox_size;
    for (int a = 0; a < 3; ++a)
      if (!std::isfinite(t_vc->translation[a])) throw StageError{VXM_EINVAL, "Ray: non-finite field"};
    const int hw = (bundle[1] - 1) / 2, hh = (bundle[2] - 1) / 2;
    for (int yi = -hh; yi <= hh; ++yi) {
      for (int xi = -hw; xi <= hw; ++xi) {
        const double v[3] = {xi * vs, yi * vs, bundle[0] * vs};
        bool zero = true;
        for (int a = 0; a < 3; ++a) {
          double d = t_vc->rotation[3 * a] * v[0];
          d = d + t_vc->rotation[3 * a + 1] * v[1];
          d = d + t_vc->rotation[3 * a + 2] * v[2];
          if (!std::isfinite(d)) throw StageError{VXM_EINVAL, "Ray: non-finite field"};
          if (d != 0.0) zero = false;
        }
        if (zero) throw StageError{VXM_EINVAL, "Ray: direction must be non-zero"};
      }
    }
    vxm::KParams kp = grid_params(*grid);
    const long long N = kp.n;
    kp.ray_vs = ray_vox_size;
    kp.vd = bundle[0];
    kp.vw = bundle[1];
    kp.vh = bundle[2];
    kp.tiles_x = (kp.vw + 7) / 8;
    kp.tiles_y = (kp.vh + 3) / 4;
    DevBuf<uint8_t> d_ms(N), d_occ(N);
    DevBuf<uint32_t> d_key(N);
    DevBuf<vxm::Counters> d_cnt(1);
    DevBuf<vxm::FrameParams> d_frame(1);
    vxm::FrameParams f{};
    fill_pose(f, *t_vc);
    vxm::set_ray_consts(f, kp.vs);
    f.epoch = kEpoch;
    f.occ_s = d_occ.p;
    f.key_s = d_key.p;
    VXM_SCK(cudaMemcpy(d_frame.p, &f, sizeof(f), cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemcpy(d_ms.p, ms, N, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemset(d_cnt.p, 0, sizeof(vxm::Counters)));
    vxm::encode_ms_kernel<<<blocks_for(N, 256), 256>>>(d_ms.p, d_occ.p, d_key.p, N, kEpoch, fmt);
    kp.occ = d_occ.p;
    kp.key = d_key.p;
    kp.key_fmt = fmt;
    kp.counters = d_cnt.p;
    kp.frames = d_frame.p;
    vxm::launch_trace(kp, 1, 1, 0);
    VXM_SCK(cudaGetLastError());
    vxm::fold_trace_slots_kernel<<<1, 32>>>(d_cnt.p);
    vxm::decode_ms_kernel<<<blocks_for(N, 256), 256>>>(d_occ.p, d_key.p, d_ms.p, N, kEpoch, fmt);
    VXM_SCK(cudaGetLastError());
    vxm::Counters cnt{};
    VXM_SCK(cudaMemcpy(&cnt, d_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost));
    VXM_SCK(cudaMemcpy(ms, d_ms.p, N, cudaMemcpyDeviceToHost));
    if (st) {
      st->rays_traced = cnt.rays_traced;
      st->voxels_freed = cnt.voxels_freed;
      st->voxels_marked_unknown_traced = cnt.voxels_traced;
      st->voxels_skipped_out_of_bounds = cnt.voxels_skipped;
    }
  });
}

int vxm_merge_grids(uint8_t* local, const uint8_t* measurement, size_t n) {
  return stage_guard([&] {
    if (n == 0) return;
    if (!local || !measurement) throw StageError{VXM_EINVAL, "null argument"};
    DevBuf<uint8_t> d(2 * n);
    VXM_SCK(cudaMemcpy(d.p, local, n, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemcpy(d.p + n, measurement, n, cudaMemcpyHostToDevice));
    // second buffer starts at offset n: vector path only when n % 16 == 0
    vxm::merge_bytes_kernel<<<blocks_for(static_cast<long long>((n + 15) / 16), 256), 256>>>(
        d.p, d.p + n, static_cast<long long>(n));
    VXM_SCK(cudaGetLastError());
    VXM_SCK(cudaMemcpy(local, d.p, n, cudaMemcpyDeviceToHost));
  });
}

int vxm_shift_grid(const int32_t dims[3], const uint8_t* in, uint8_t* out, const int32_t offset[3]) {
  return stage_guard([&] {
    if (!dims || !in || !out || !offset) throw StageError{VXM_EINVAL, "null argument"};
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1) throw StageError{VXM_EINVAL, "empty grid"};
    const long long N = static_cast<long long>(dims[0]) * dims[1] * dims[2];
    DevBuf<uint8_t> d(2 * N);
    VXM_SCK(cudaMemcpy(d.p, in, N, cudaMemcpyHostToDevice));
    vxm::shift_kernel<<<blocks_for(N, 256), 256>>>(d.p, d.p + N, dims[0], dims[1], dims[2],
                                                   offset[0], offset[1], offset[2]);
    VXM_SCK(cudaGetLastError());
    VXM_SCK(cudaMemcpy(out, d.p + N, N, cudaMemcpyDeviceToHost));
  });
}

int vxm_depth_to_cloud(const vxm_camera* cam, const float* depth, double* xs, double* ys,
                       double* zs, size_t* n_out) {
  return stage_guard([&] {
    if (!cam || !depth || !n_out) throw StageError{VXM_EINVAL, "null argument"};
    // CameraModel::validate (geometry.cpp:28-41)
    const double pi = 3.14159265358979323846;
    if (cam->width <= 0 || cam->height <= 0)
      throw StageError{VXM_EINVAL, "CameraModel: width and height must be positive"};
    if (!(cam->fov_x > 0.0) || !(cam->fov_x < pi) || !(cam->fov_y > 0.0) || !(cam->fov_y < pi))
      throw StageError{VXM_EINVAL, "CameraModel: FOV must lie in (0, pi)"};
    if (!(cam->max_depth > 0.0) || !std::isfinite(cam->max_depth))
      throw StageError{VXM_EINVAL, "CameraModel: max_depth must be positive and finite"};
    const int W = cam->width, H = cam->height;
    const size_t npix = static_cast<size_t>(W) * H;
    DevBuf<float> d_depth(npix);
    DevBuf<unsigned> d_rows(H);
    DevBuf<unsigned long long> d_off(H + 1);
    DevBuf<double> d_pts(3 * npix);
    VXM_SCK(cudaMemcpy(d_depth.p, depth, sizeof(float) * npix, cudaMemcpyHostToDevice));
    const double fx = (W / 2.0) / std::tan(cam->fov_x / 2.0);
    const double fy = (H / 2.0) / std::tan(cam->fov_y / 2.0);
    vxm::cloud_count_rows_kernel<<<H, 256>>>(d_depth.p, W, cam->max_depth, d_rows.p);
    vxm::cloud_scan_rows_kernel<<<1, 32>>>(d_rows.p, d_off.p, H);
    vxm::cloud_write_rows_kernel<<<H, 256>>>(d_depth.p, W, fx, fy, W / 2.0, H / 2.0,
                                             cam->max_depth, d_off.p, d_pts.p, d_pts.p + npix,
                                             d_pts.p + 2 * npix);
    VXM_SCK(cudaGetLastError());
    unsigned long long total = 0;
    VXM_SCK(cudaMemcpy(&total, d_off.p + H, sizeof(total), cudaMemcpyDeviceToHost));
    *n_out = static_cast<size_t>(total);
    if (total) {
      if (!xs || !ys || !zs) throw StageError{VXM_EINVAL, "null cloud arrays"};
      VXM_SCK(cudaMemcpy(xs, d_pts.p, sizeof(double) * total, cudaMemcpyDeviceToHost));
      VXM_SCK(cudaMemcpy(ys, d_pts.p + npix, sizeof(double) * total, cudaMemcpyDeviceToHost));
      VXM_SCK(cudaMemcpy(zs, d_pts.p + 2 * npix, sizeof(double) * total, cudaMemcpyDeviceToHost));
    }
  });
}

// sim::render_depth for n_frames poses. out: HOST or DEVICE
// memory of n_frames * width * height floats.
int vxm_render_depth(const vxm_camera* cam, const vxm_pose* t_wc, int32_t n_frames, const double* boxes,
                     int32_t n_boxes, float* out, int32_t device) {
  return stage_guard([&] {
    int count = 0;
    VXM_SCK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw StageError{VXM_EINVAL, "device index out of range"};
    VXM_SCK(cudaSetDevice(device));
    if (!cam || !t_wc || !out || (n_boxes > 0 && !boxes)) throw StageError{VXM_EINVAL, "null argument"};
    if (n_frames < 1 || n_boxes < 0) throw StageError{VXM_EINVAL, "n_frames must be >= 1, n_boxes >= 0"};
    // CameraModel::validate (geometry.cpp:28-41) and Aabb::validate (scene.cpp:12-17)
    const double pi = 3.14159265358979323846;
    if (cam->width <= 0 || cam->height <= 0)
      throw StageError{VXM_EINVAL, "CameraModel: width and height must be positive"};
    if (!(cam->fov_x > 0.0) || !(cam->fov_x < pi) || !(cam->fov_y > 0.0) || !(cam->fov_y < pi))
      throw StageError{VXM_EINVAL, "CameraModel: FOV must lie in (0, pi)"};
    if (!(cam->max_depth > 0.0) || !std::isfinite(cam->max_depth))
      throw StageError{VXM_EINVAL, "CameraModel: max_depth must be positive and finite"};
    for (int b = 0; b < n_boxes; ++b)
      for (int a = 0; a < 3; ++a) {
        const double lo = boxes[6 * b + a], hi = boxes[6 * b + 3 + a];
        if (!std::isfinite(lo) || !std::isfinite(hi) || !(lo < hi))
          throw StageError{VXM_EINVAL, "Aabb: min must be strictly below max on every axis"};
      }
    const int W = cam->width, H = cam->height;
    const size_t npix = static_cast<size_t>(W) * H;
    // ((u + 0.5) - cx) / fx per column, likewise per row (render.cpp:30-41)
    const double fx = (W / 2.0) / std::tan(cam->fov_x / 2.0);
    const double fy = (H / 2.0) / std::tan(cam->fov_y / 2.0);
    std::vector<double> q(static_cast<size_t>(W) + H);
    for (int u = 0; u < W; ++u) q[u] = ((u + 0.5) - W / 2.0) / fx;
    for (int v = 0; v < H; ++v) q[W + v] = ((v + 0.5) - H / 2.0) / fy;
    std::vector<double> P(12 * static_cast<size_t>(n_frames));
    for (int f = 0; f < n_frames; ++f) {
      for (int i = 0; i < 9; ++i) P[12 * f + i] = t_wc[f].rotation[i];
      for (int i = 0; i < 3; ++i) P[12 * f + 9 + i] = t_wc[f].translation[i];
    }
    DevBuf<double> d_q(q.size()), d_p(P.size()), d_b(6 * static_cast<size_t>(n_boxes) + 1);
    VXM_SCK(cudaMemcpy(d_q.p, q.data(), sizeof(double) * q.size(), cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemcpy(d_p.p, P.data(), sizeof(double) * P.size(), cudaMemcpyHostToDevice));
    if (n_boxes) VXM_SCK(cudaMemcpy(d_b.p, boxes, sizeof(double) * 6 * n_boxes, cudaMemcpyHostToDevice));
    cudaPointerAttributes attr{};
    const bool dev_out = cudaPointerGetAttributes(&attr, out) == cudaSuccess && attr.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    DevBuf<float> d_out(dev_out ? 0 : npix * n_frames);
    float* dst = dev_out ? out : d_out.p;
    const size_t smem = n_boxes <= 1024 ? sizeof(double) * 6 * n_boxes : 0;
    vxm::render_depth_kernel<<<dim3(static_cast<unsigned>((npix + 255) / 256), n_frames), 256, smem>>>(
        d_q.p, W, H, cam->max_depth, d_p.p, d_b.p, n_boxes, dst);
    VXM_SCK(cudaGetLastError());
    if (dev_out) {
      VXM_SCK(cudaDeviceSynchronize());
    } else {
      VXM_SCK(cudaMemcpy(out, d_out.p, sizeof(float) * npix * n_frames, cudaMemcpyDeviceToHost));
    }
  });
}

// KernelTable adapter. The reference signatures are void with no error
// channel, so a failure here is fatal and loud.
static void adapter_fail(const char* what) {
  std::fprintf(stderr, "vxm kernel adapter: %s\n", what);
  std::abort();
}

void vxm_kernel_merge(uint8_t* local, const uint8_t* measurement, size_t n) {
  if (vxm_merge_grids(local, measurement, n) != VXM_OK) adapter_fail(vxm_last_error());
}

void vxm_kernel_transform_voxelize(const double* xs, const double* ys, const double* zs,
                                   size_t n, const double* rotation, const double* translation,
                                   double vox_size, int32_t* cx, int32_t* cy, int32_t* cz) {
  if (n == 0) return;
  const int rc = stage_guard([&] {
    DevBuf<double> d_in(3 * n + 12);
    DevBuf<int32_t> d_out(3 * n);
    VXM_SCK(cudaMemcpy(d_in.p, xs, sizeof(double) * n, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemcpy(d_in.p + n, ys, sizeof(double) * n, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemcpy(d_in.p + 2 * n, zs, sizeof(double) * n, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemcpy(d_in.p + 3 * n, rotation, sizeof(double) * 9, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemcpy(d_in.p + 3 * n + 9, translation, sizeof(double) * 3, cudaMemcpyHostToDevice));
    vxm::transform_voxelize_kernel<<<blocks_for(static_cast<long long>(n), 256), 256>>>(
        d_in.p, d_in.p + n, d_in.p + 2 * n, static_cast<long long>(n), d_in.p + 3 * n,
        d_in.p + 3 * n + 9, vox_size, d_out.p, d_out.p + n, d_out.p + 2 * n);
    VXM_SCK(cudaGetLastError());
    VXM_SCK(cudaMemcpy(cx, d_out.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    VXM_SCK(cudaMemcpy(cy, d_out.p + n, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    VXM_SCK(cudaMemcpy(cz, d_out.p + 2 * n, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  });
  if (rc != VXM_OK) adapter_fail(vxm_last_error());
}

const char* vxm_kernel_isa(void) { return "cuda-sm100a"; }

int vxm_trace_per_pixel(const vxm_grid_spec* grid, uint8_t* ms, const double* xs,
                        const double* ys, const double* zs, size_t n, const vxm_pose* t_vc,
                        vxm_trace_stats* st) {
  return stage_guard([&] {
    check_grid(grid);
    if (!ms || !t_vc || (n && (!xs || !ys || !zs))) throw StageError{VXM_EINVAL, "null argument"};
    // world_to_voxel of the camera centre throws on non-finite input (grid.cpp:54-57)
    for (int a = 0; a < 3; ++a)
      if (!std::isfinite(t_vc->translation[a]))
        throw StageError{VXM_EINVAL, "world_to_voxel: non-finite point"};
    vxm::KParams kp = grid_params(*grid);
    const long long N = kp.n;
    DevBuf<uint8_t> d_ms(N), d_occ(N);
    DevBuf<uint32_t> d_key(N);
    DevBuf<double> d_pts(3 * n + 1);
    DevBuf<vxm::Counters> d_cnt(1);
    DevBuf<vxm::FrameParams> d_frame(1);
    vxm::FrameParams f{};
    fill_pose(f, *t_vc);
    f.xs = d_pts.p;
    f.ys = d_pts.p + n;
    f.zs = d_pts.p + 2 * n;
    f.n_points = static_cast<long long>(n);
    f.epoch = kEpoch;
    VXM_SCK(cudaMemcpy(d_frame.p, &f, sizeof(f), cudaMemcpyHostToDevice));
    if (n) {
      VXM_SCK(cudaMemcpy(d_pts.p, xs, sizeof(double) * n, cudaMemcpyHostToDevice));
      VXM_SCK(cudaMemcpy(d_pts.p + n, ys, sizeof(double) * n, cudaMemcpyHostToDevice));
      VXM_SCK(cudaMemcpy(d_pts.p + 2 * n, zs, sizeof(double) * n, cudaMemcpyHostToDevice));
    }
    VXM_SCK(cudaMemcpy(d_ms.p, ms, N, cudaMemcpyHostToDevice));
    VXM_SCK(cudaMemset(d_cnt.p, 0, sizeof(vxm::Counters)));
    vxm::encode_ms_kernel<<<blocks_for(N, 256), 256>>>(d_ms.p, d_occ.p, d_key.p, N, kEpoch, vxm::kEpochKeys);
    kp.occ = d_occ.p;
    kp.key = d_key.p;
    kp.key_fmt = vxm::kEpochKeys;
    kp.counters = d_cnt.p;
    kp.frames = d_frame.p;
    vxm::trace_per_pixel_kernel<<<dim3(blocks_for(static_cast<long long>(n), 256), 1), 256>>>(kp, 0);
    VXM_SCK(cudaGetLastError());
    vxm::fold_trace_slots_kernel<<<1, 32>>>(d_cnt.p);
    vxm::decode_ms_kernel<<<blocks_for(N, 256), 256>>>(d_occ.p, d_key.p, d_ms.p, N, kEpoch, vxm::kEpochKeys);
    VXM_SCK(cudaGetLastError());
    vxm::Counters cnt{};
    VXM_SCK(cudaMemcpy(&cnt, d_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost));
    VXM_SCK(cudaMemcpy(ms, d_ms.p, N, cudaMemcpyDeviceToHost));
    if (st) {
      st->rays_traced = cnt.rays_traced;
      st->voxels_freed = cnt.voxels_freed;
      st->voxels_marked_unknown_traced = cnt.voxels_traced;
      st->voxels_skipped_out_of_bounds = cnt.voxels_skipped;
    }
  });
}

}  // extern "C"
