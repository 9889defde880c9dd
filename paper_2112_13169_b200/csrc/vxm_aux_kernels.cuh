// Kernels behind the stand-alone entry points of the public API (host grids
// in, host grids out): byte <-> word conversion of measurement grids, the
// KernelTable merge / transform_voxelize adapters, shift_grid_by, and the
// ordered compaction of depth_to_cloud.
#pragma once

#include "vxm_device.cuh"
#include "vxm_kernels.cuh"

namespace vxm {

// Reference byte grid -> (occ, keys) of epoch e (see vxm_device.cuh):
// Occupied becomes occ == e (and, clear format, the Occupied key);
// pre-existing Free / UnknownTraced become the lowest-priority keys so that
// any ray write overrides them.
__global__ void encode_ms_kernel(const uint8_t* ms, uint8_t* occ, uint32_t* key, long long n, uint32_t epoch,
                                 int fmt) {
  const uint32_t carried = ray_key(fmt, epoch, -1);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint8_t b = ms[i];
    occ[i] = b == 2 ? static_cast<uint8_t>(epoch) : 0;
    key[i] = (b == 1 || b == 3) ? (carried | (b >> 1)) : (b == 2 && fmt == kClearKeys ? kClearOccupied : 0u);
  }
}

// (occ, keys) -> reference bytes. keep_input (populate, which only adds
// Occupied cells): every cell not Occupied now keeps its input byte (the
// vectorised dilation may store Unknown next to the cells it marks).
__global__ void decode_ms_kernel(const uint8_t* occ, const uint32_t* key, uint8_t* ms, long long n, uint32_t epoch,
                                 int fmt, int keep_input = 0) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint32_t v = fmt == kClearKeys ? decode_clear_key(key[i]) : decode_cell(occ[i], key[i], epoch);
    ms[i] = static_cast<uint8_t>(keep_input && v != 2u ? ms[i] : v);
  }
}

// MergeFn over raw bytes (kernels_scalar.cpp:10-16), 16 cells per thread
// when the pointers allow 16-byte vectors.
__global__ void merge_bytes_kernel(uint8_t* local, const uint8_t* ms, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(local) | reinterpret_cast<uintptr_t>(ms)) & 15u) == 0;
  const long long nvec = vec ? n / 16 : 0;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < nvec;
       q += stride) {
    uint4 l = reinterpret_cast<uint4*>(local)[q];
    const uint4 m = reinterpret_cast<const uint4*>(ms)[q];
    uint32_t* lw = reinterpret_cast<uint32_t*>(&l);
    const uint32_t* mw = reinterpret_cast<const uint32_t*>(&m);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t out = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        out |= merge_cell((lw[w] >> (8 * b)) & 0xffu, (mw[w] >> (8 * b)) & 0xffu) << (8 * b);
      }
      lw[w] = out;
    }
    reinterpret_cast<uint4*>(local)[q] = l;
  }
  for (long long i = nvec * 16 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       i < n; i += stride) {
    local[i] = static_cast<uint8_t>(merge_cell(local[i], ms[i]));
  }
}

// TransformVoxelizeFn (kernels_scalar.cpp:18-37), one point per thread.
__global__ void transform_voxelize_kernel(const double* xs, const double* ys, const double* zs,
                                          long long n, const double* R, const double* t,
                                          double vs, int32_t* cx, int32_t* cy, int32_t* cz) {
  double Rr[9], tt[3];
  const double inv_vs = __drcp_rn(vs);
#pragma unroll
  for (int i = 0; i < 9; ++i) Rr[i] = R[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) tt[i] = t[i];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int c[3];
    transform_voxelize(Rr, tt, xs[i], ys[i], zs[i], vs, inv_vs, c);
    cx[i] = c[0];
    cy[i] = c[1];
    cz[i] = c[2];
  }
}

// shift_grid_by (grid.cpp:81-108) as a gather.
__global__ void shift_kernel(const uint8_t* in, uint8_t* out, int dx, int dy, int dz, int ox,
                             int oy, int oz) {
  const long long n = static_cast<long long>(dx) * dy * dz;
  const long long dxy = static_cast<long long>(dx) * dy;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int z = static_cast<int>(c / dxy);
    const long long rem = c - z * dxy;
    const int y = static_cast<int>(rem / dx);
    const int x = static_cast<int>(rem - static_cast<long long>(y) * dx);
    const int sx = x + ox, sy = y + oy, sz = z + oz;
    uint8_t v = 0;
    if (sx >= 0 && sy >= 0 && sz >= 0 && sx < dx && sy < dy && sz < dz) {
      v = in[sx + static_cast<long long>(sy) * dx + static_cast<long long>(sz) * dxy];
    }
    out[c] = v;
  }
}

// depth_to_cloud: row-major order of valid pixels is the output order in both
// reference execution modes (geometry.cpp:79-97). Pass 1 counts valid pixels
// per row, pass 2 scans the row counts, pass 3 writes each row's points at
// its offset with an in-block ordered scan.
__device__ __forceinline__ bool pixel_valid(float d, double max_depth) {
  return isfinite(d) && d > 0.0f && !(static_cast<double>(d) > max_depth);
}

__global__ void cloud_count_rows_kernel(const float* depth, int W, double max_depth,
                                        unsigned* row_count) {
  const int v = blockIdx.x;
  unsigned c = 0;
  for (int u = threadIdx.x; u < W; u += blockDim.x) c += pixel_valid(depth[static_cast<long long>(v) * W + u], max_depth);
  unsigned vals[1] = {c};
  __shared__ unsigned long long acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  unsigned long long* dst[1] = {&acc};
  block_accumulate<1>(vals, dst);
  __syncthreads();
  if (threadIdx.x == 0) row_count[v] = static_cast<unsigned>(acc);
}

__global__ void cloud_scan_rows_kernel(const unsigned* row_count, unsigned long long* row_off,
                                       int H) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long run = 0;
    for (int v = 0; v < H; ++v) {
      row_off[v] = run;
      run += row_count[v];
    }
    row_off[H] = run;
  }
}

__global__ void __launch_bounds__(256) cloud_write_rows_kernel(const float* depth, int W,
                                                               double fx, double fy, double cx,
                                                               double cy, double max_depth,
                                                               const unsigned long long* row_off,
                                                               double* xs, double* ys,
                                                               double* zs) {
  __shared__ unsigned warp_tot[8];
  const int v = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long base = row_off[v];
  for (int u0 = 0; u0 < W; u0 += blockDim.x) {
    const int u = u0 + threadIdx.x;
    const float d = u < W ? depth[static_cast<long long>(v) * W + u] : 0.0f;
    const bool ok = u < W && pixel_valid(d, max_depth);
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    const unsigned before = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    unsigned woff = 0, total = 0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) {
      if (w < warp) woff += warp_tot[w];
      total += warp_tot[w];
    }
    if (ok) {
      const double D = static_cast<double>(d);
      const unsigned long long o = base + woff + before;
      xs[o] = dmul(ddiv(dsub(dadd(static_cast<double>(u), 0.5), cx), fx), D);
      ys[o] = dmul(ddiv(dsub(dadd(static_cast<double>(v), 0.5), cy), fy), D);
      zs[o] = D;
    }
    base += total;
    __syncthreads();
  }
}

// Stand-alone trace: fold K3's slots (K4 does this in the per-frame graph).
__global__ void fold_trace_slots_kernel(Counters* c) { fold_trace_slots(*c); }

// ---------------------------------------------------------------------------
// sim::render_depth (proj/src/sim/render.cpp:26-58) with ray_box_hit
// (render.cpp:8-24): one thread per pixel, a block row of frames per
// blockIdx.y. dir = R * ((u+0.5-cx)/fx, (v+0.5-cy)/fy, 1) with left-to-right
// row sums (the Eigen subset's order), slab test per box with IEEE
// divisions and std::max/std::min comparison semantics, nearest s > 0,
// depth = (float)s when s <= max_depth, else the invalid sentinel 0.
// boxes: nb x (minx miny minz maxx maxy maxz); poses: 12 doubles per frame
// (R row-major, t).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) render_depth_kernel(const double* qtab, int W, int H, double max_depth,
                                                           const double* poses, const double* boxes, int nb,
                                                           float* out) {
  extern __shared__ double sbox[];
  const bool in_smem = nb <= 1024;
  if (in_smem)
    for (int i = threadIdx.x; i < 6 * nb; i += blockDim.x) sbox[i] = boxes[i];
  __syncthreads();
  const double* bx = in_smem ? sbox : boxes;
  const int f = blockIdx.y;
  const long long npix = static_cast<long long>(W) * H;
  const long long pix = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pix >= npix) return;
  const int v = static_cast<int>(pix / W), u = static_cast<int>(pix - static_cast<long long>(v) * W);
  const double* P = poses + 12 * f;
  const double dc[3] = {qtab[u], qtab[W + v], 1.0};
  double dir[3], o[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    dir[a] = dadd(dadd(dmul(P[3 * a], dc[0]), dmul(P[3 * a + 1], dc[1])), dmul(P[3 * a + 2], dc[2]));
    o[a] = P[9 + a];
  }
  double best = __longlong_as_double(0x7ff0000000000000ll);
  for (int b = 0; b < nb; ++b) {
    const double* lo = bx + 6 * b;
    const double* hi = lo + 3;
    double t_near = -__longlong_as_double(0x7ff0000000000000ll);
    double t_far = __longlong_as_double(0x7ff0000000000000ll);
    bool miss = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (dir[a] == 0.0) {
        miss = miss || o[a] < lo[a] || o[a] > hi[a];
        continue;
      }
      double ta = ddiv(dsub(lo[a], o[a]), dir[a]);
      double tb = ddiv(dsub(hi[a], o[a]), dir[a]);
      if (ta > tb) {
        const double w = ta;
        ta = tb;
        tb = w;
      }
      t_near = t_near < ta ? ta : t_near;  // std::max(t_near, ta)
      t_far = tb < t_far ? tb : t_far;     // std::min(t_far, tb)
    }
    if (miss || t_near > t_far || t_far <= 0.0) continue;
    const double s = t_near > 0.0 ? t_near : t_far;
    if (s > 0.0 && s < best) best = s;
  }
  out[static_cast<long long>(f) * npix + pix] = best <= max_depth ? __double2float_rn(best) : 0.0f;
}

}  // namespace vxm
