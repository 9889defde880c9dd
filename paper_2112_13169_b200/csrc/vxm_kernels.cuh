// The per-frame voxelization kernels (paper Alg. 1-3 + the local-grid shift).
// One CUDA grid dimension (blockIdx.y) indexes independent sensor streams, so
// a batch of S streams is one launch per stage.
//
//   K1 populate_depth / populate_cloud   depth -> point -> T_vc -> voxel -> Occupied
//   K2 dilate                           vox_inf > 0: Chebyshev dilation of the centres
//   K3 trace_bundle                     frustum ray casting, Free / UnknownTraced
//   K4 merge_shift_count                merge into the local grid, shift, count
#pragma once

#include "vxm_device.cuh"

namespace vxm {

// ---------------------------------------------------------------------------
// K1: depth_to_cloud (proj/src/geometry.cpp:45-57) fused with
// voxelize_points + mark_point for the centre voxel (proj/src/integrator.cpp:
// 24-41, 62-85). Each thread owns 4 consecutive pixels (one 16-byte load).
// Pixels never materialise as a point cloud.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void populate_point(const KParams& p, const FrameParams& f,
                                               uint32_t* target, uint32_t occ, double x,
                                               double y, double z, unsigned& outside) {
  int c[3];
  transform_voxelize(f.rot, f.trans, x, y, z, p.vs, c);
  if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[0] >= p.dx || c[1] >= p.dy || c[2] >= p.dz) {
    ++outside;
    return;
  }
  const long long idx = static_cast<long long>(c[0]) +
                        static_cast<long long>(c[1]) * p.dx +
                        static_cast<long long>(c[2]) * p.dx * p.dy;
  target[idx] = occ;  // idempotent: every writer stores the same word
}

__device__ __forceinline__ void back_project(const KParams& p, int u, int v, double depth,
                                             double& x, double& y) {
  // x = (u + 0.5 - cx) / fx * depth  (geometry.cpp:55-56), left to right.
  x = dmul(ddiv(dsub(dadd(static_cast<double>(u), 0.5), p.cx), p.fx), depth);
  y = dmul(ddiv(dsub(dadd(static_cast<double>(v), 0.5), p.cy), p.fy), depth);
}

__global__ void __launch_bounds__(256) populate_depth_kernel(KParams p) {
  const int s = blockIdx.y;
  const FrameParams& f = p.frames[s];
  uint32_t* target = (p.vox_inf > 0 ? p.ctr : p.msw) + static_cast<long long>(s) * p.n;
  const uint32_t occ = occupied_word(f.tag);
  const long long npix = static_cast<long long>(p.W) * p.H;
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long first = q * 4;

  unsigned total = 0, outside = 0;
  if (first < npix) {
    float d[4];
    if (first + 3 < npix && ((reinterpret_cast<uintptr_t>(f.depth) & 15u) == 0)) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(f.depth) + q);
      d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) d[i] = first + i < npix ? f.depth[first + i] : 0.0f;
    }
    const int v0 = static_cast<int>(first / p.W);
    const int u0 = static_cast<int>(first - static_cast<long long>(v0) * p.W);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int u = u0 + i, v = v0;
      if (u >= p.W) { u -= p.W; ++v; }
      const float di = d[i];
      // DepthImage::valid_depth (geometry.hpp:124): finite and > 0; then the
      // max-depth cut on the promoted double (geometry.cpp:53-54).
      if (!(isfinite(di) && di > 0.0f)) continue;
      const double depth = static_cast<double>(di);
      if (depth > p.max_depth) continue;
      ++total;
      double x, y;
      back_project(p, u, v, depth, x, y);
      populate_point(p, f, target, occ, x, y, depth, outside);
    }
  }
  unsigned vals[2] = {total, outside};
  unsigned long long* dst[2] = {&p.counters[s].points_total, &p.counters[s].points_outside};
  block_accumulate<2>(vals, dst);
}

// K1 for an explicit camera-frame cloud (MeasurementFrame::cloud). Points
// that PointCloud::add would have dropped (non-finite) are skipped uncounted
// (proj/include/voxmap/geometry.hpp:84-89).
__global__ void __launch_bounds__(256) populate_cloud_kernel(KParams p) {
  const int s = blockIdx.y;
  const FrameParams& f = p.frames[s];
  uint32_t* target = (p.vox_inf > 0 ? p.ctr : p.msw) + static_cast<long long>(s) * p.n;
  const uint32_t occ = occupied_word(f.tag);
  unsigned total = 0, outside = 0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < f.n_points; i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double x = f.xs[i], y = f.ys[i], z = f.zs[i];
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) continue;
    ++total;
    populate_point(p, f, target, occ, x, y, z, outside);
  }
  unsigned vals[2] = {total, outside};
  unsigned long long* dst[2] = {&p.counters[s].points_total, &p.counters[s].points_outside};
  block_accumulate<2>(vals, dst);
}

// ---------------------------------------------------------------------------
// K2: obstacle inflation. mark_point writes the (2r+1)^3 cube around every
// in-bounds centre, clipped to the grid (integrator.cpp:70-83); that is a
// Chebyshev dilation of the centre set restricted to the grid, which is
// separable: three 1-D max filters. One block produces a 32x8x8 tile from a
// shared-memory copy of the tile plus an r-voxel halo.
// ---------------------------------------------------------------------------
constexpr int kDilTX = 32, kDilTY = 8, kDilTZ = 8;

__global__ void __launch_bounds__(256) dilate_kernel(KParams p, int r) {
  extern __shared__ uint8_t smem[];
  const int s = blockIdx.z;
  const FrameParams& f = p.frames[s];
  const uint32_t occ = occupied_word(f.tag);
  const uint32_t* ctr = p.ctr + static_cast<long long>(s) * p.n;
  uint32_t* msw = p.msw + static_cast<long long>(s) * p.n;

  const int tiles_x = (p.dx + kDilTX - 1) / kDilTX;
  const int x0 = (blockIdx.x % tiles_x) * kDilTX;
  const int y0 = (blockIdx.x / tiles_x) * kDilTY;
  const int z0 = blockIdx.y * kDilTZ;
  const int HX = kDilTX + 2 * r, HY = kDilTY + 2 * r, HZ = kDilTZ + 2 * r;
  uint8_t* in = smem;                       // HZ x HY x HX
  uint8_t* tx = in + HX * HY * HZ;          // HZ x HY x TX
  uint8_t* ty = tx + kDilTX * HY * HZ;      // HZ x TY x TX
  const int tid = threadIdx.x;

  for (int i = tid; i < HX * HY * HZ; i += blockDim.x) {
    const int hx = i % HX, hy = (i / HX) % HY, hz = i / (HX * HY);
    const int x = x0 - r + hx, y = y0 - r + hy, z = z0 - r + hz;
    uint8_t c = 0;
    if (x >= 0 && y >= 0 && z >= 0 && x < p.dx && y < p.dy && z < p.dz) {
      const long long idx = x + static_cast<long long>(y) * p.dx +
                            static_cast<long long>(z) * p.dx * p.dy;
      c = ctr[idx] == occ;
    }
    in[i] = c;
  }
  __syncthreads();
  for (int i = tid; i < kDilTX * HY * HZ; i += blockDim.x) {
    const int x = i % kDilTX, yz = i / kDilTX;
    const uint8_t* row = in + yz * HX + x;
    uint8_t m = 0;
    for (int k = 0; k <= 2 * r; ++k) m |= row[k];
    tx[i] = m;
  }
  __syncthreads();
  for (int i = tid; i < kDilTX * kDilTY * HZ; i += blockDim.x) {
    const int x = i % kDilTX, y = (i / kDilTX) % kDilTY, z = i / (kDilTX * kDilTY);
    const uint8_t* col = tx + (z * HY + y) * kDilTX + x;
    uint8_t m = 0;
    for (int k = 0; k <= 2 * r; ++k) m |= col[k * kDilTX];
    ty[i] = m;
  }
  __syncthreads();
  for (int i = tid; i < kDilTX * kDilTY * kDilTZ; i += blockDim.x) {
    const int x = i % kDilTX, y = (i / kDilTX) % kDilTY, z = i / (kDilTX * kDilTY);
    const int gx = x0 + x, gy = y0 + y, gz = z0 + z;
    if (gx >= p.dx || gy >= p.dy || gz >= p.dz) continue;
    const uint8_t* col = ty + z * kDilTY * kDilTX + y * kDilTX + x;
    uint8_t m = 0;
    for (int k = 0; k <= 2 * r; ++k) m |= col[k * kDilTY * kDilTX];
    if (m) {
      msw[gx + static_cast<long long>(gy) * p.dx + static_cast<long long>(gz) * p.dx * p.dy] = occ;
    }
  }
}

// ---------------------------------------------------------------------------
// K3: bundled frustum ray casting (paper Alg. 2): generate_rays
// (proj/src/raytracer.cpp:35-61) + walk_ray (proj/include/voxmap/raytracer.hpp:
// 76-118) + traverse_ray (raytracer.cpp:63-96). One thread per ray; a warp
// owns an 8x4 tile of end-plane targets so that its rays stay spatially
// coherent. The Sequential last-writer rule becomes atomicMax on the cell
// word (see vxm_device.cuh); before issuing it a lane drops its write when
// lane+1 or lane+8 (both higher ray indices) writes the same cell in the same
// step, which removes most same-address traffic near the camera.
// ---------------------------------------------------------------------------
struct RayState {
  int cur[3];
  int step[3];
  double tmax[3];
  double tdelta[3];
  double stop;  // max_dist - kTraversalStopEpsilon
};

// One ray's setup, operation for operation as generate_rays + walk_ray.
// dir = R * (xi*vs, yi*vs, vd*vs) with left-to-right row sums (the Eigen
// subset's order; every order agrees for the axis-aligned poses used by the
// golden vectors), |dir|^2 = (d0^2 + d1^2) + d2^2 (Eigen's vectorized redux).
__device__ __forceinline__ void ray_setup(const double* R, const double* start, double vs,
                                          int xi, int yi, int vd, RayState& st) {
  const double v0 = dmul(static_cast<double>(xi), vs);
  const double v1 = dmul(static_cast<double>(yi), vs);
  const double v2 = dmul(static_cast<double>(vd), vs);
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    d[a] = dadd(dadd(dmul(R[3 * a], v0), dmul(R[3 * a + 1], v1)), dmul(R[3 * a + 2], v2));
  }
  const double xs = static_cast<double>(xi), ys = static_cast<double>(yi),
               ds = static_cast<double>(vd);
  const double max_dist = dmul(vs, __dsqrt_rn(dadd(dadd(dmul(xs, xs), dmul(ys, ys)), dmul(ds, ds))));
  st.stop = dsub(max_dist, 1e-10);
  const double n2 = dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2]));
  const double nrm = __dsqrt_rn(n2);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double u = n2 > 0.0 ? ddiv(d[a], nrm) : d[a];
    st.cur[a] = static_cast<int>(floor(ddiv(start[a], vs)));
    if (u > 0.0) {
      st.step[a] = 1;
      st.tmax[a] = ddiv(dsub(dmul(static_cast<double>(st.cur[a] + 1), vs), start[a]), u);
      st.tdelta[a] = ddiv(vs, u);
    } else if (u < 0.0) {
      st.step[a] = -1;
      st.tmax[a] = ddiv(dsub(dmul(static_cast<double>(st.cur[a]), vs), start[a]), u);
      st.tdelta[a] = ddiv(vs, -u);
    } else {
      st.step[a] = 0;
      st.tmax[a] = __longlong_as_double(0x7ff0000000000000ll);
      st.tdelta[a] = st.tmax[a];
    }
  }
}

__global__ void __launch_bounds__(128) trace_bundle_kernel(KParams p) {
  const int s = blockIdx.y;
  const FrameParams& f = p.frames[s];
  uint32_t* msw = p.msw + static_cast<long long>(s) * p.n;
  const uint32_t occ = occupied_word(f.tag);

  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
  const int xi_idx = tx * 8 + (lane & 7);
  const int yi_idx = ty * 4 + (lane >> 3);
  const bool active = ty < p.tiles_y && xi_idx < p.vw && yi_idx < p.vh;

  const int hw = (p.vw - 1) / 2, hh = (p.vh - 1) / 2;
  const uint32_t ray = static_cast<uint32_t>(yi_idx) * p.vw + xi_idx;  // row-major, y outer
  RayState st;
  ray_setup(f.rot, f.trans, p.vs, xi_idx - hw, yi_idx - hh, p.vd, st);

  bool alive = active;
  bool entered = false;
  uint32_t traced_bit = 0;
  unsigned freed = 0, traced = 0, skipped = 0;
  const long long dxy = static_cast<long long>(p.dx) * p.dy;

  while (__any_sync(0xffffffffu, alive)) {
    bool write = false;
    uint32_t idx = 0xffffffffu - lane;  // unique non-cell sentinel for idle lanes
    if (alive) {
      const int x = st.cur[0], y = st.cur[1], z = st.cur[2];
      if (x < 0 || y < 0 || z < 0 || x >= p.dx || y >= p.dy || z >= p.dz) {
        if (entered) {
          alive = false;  // a line leaves a convex grid exactly once
        } else {
          ++skipped;
        }
      } else {
        entered = true;
        const uint32_t cell = static_cast<uint32_t>(x + y * p.dx + z * dxy);
        if (msw[cell] == occ) {
          traced_bit = 1;
        } else {
          write = true;
          idx = cell;
          if (traced_bit) ++traced; else ++freed;
        }
      }
    }
    const uint32_t right = __shfl_down_sync(0xffffffffu, idx, 1);
    const uint32_t below = __shfl_down_sync(0xffffffffu, idx, 8);
    const bool dominated = (lane < 31 && right == idx) || (lane < 24 && below == idx);
    if (write && !dominated) {
      atomicMax(msw + idx, f.tag | ((ray + 1u) << 1) | traced_bit);
    }
    if (alive) {
      int axis;
      if (st.tmax[0] <= st.tmax[1] && st.tmax[0] <= st.tmax[2]) {
        axis = 0;
      } else if (st.tmax[1] <= st.tmax[2]) {
        axis = 1;
      } else {
        axis = 2;
      }
      const double tm = axis == 0 ? st.tmax[0] : (axis == 1 ? st.tmax[1] : st.tmax[2]);
      if (tm >= st.stop) {
        alive = false;
      } else {
        if (axis == 0) { st.cur[0] += st.step[0]; st.tmax[0] = dadd(st.tmax[0], st.tdelta[0]); }
        else if (axis == 1) { st.cur[1] += st.step[1]; st.tmax[1] = dadd(st.tmax[1], st.tdelta[1]); }
        else { st.cur[2] += st.step[2]; st.tmax[2] = dadd(st.tmax[2], st.tdelta[2]); }
      }
    }
  }
  unsigned vals[4] = {active ? 1u : 0u, freed, traced, skipped};
  unsigned long long* dst[4] = {&p.counters[s].rays_traced, &p.counters[s].voxels_freed,
                                &p.counters[s].voxels_traced, &p.counters[s].voxels_skipped};
  block_accumulate<4>(vals, dst);
}

// ---------------------------------------------------------------------------
// K4: merge_grids (proj/src/pipeline.cpp:44-61) + shift_grid_by
// (proj/src/grid.cpp:81-108) + the two VoxelGrid::count passes
// (pipeline.cpp:114-115) in one gather: destination cell c takes
// merge(loc[c+off], ms[c+off]) when c+off is inside the grid, else Unknown.
// Reads the current local buffer, writes the other (ping-pong). Each thread
// produces 4 consecutive cells (one 32-bit store).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) merge_shift_count_kernel(KParams p) {
  const int s = blockIdx.y;
  const FrameParams& f = p.frames[s];
  const long long base = static_cast<long long>(s) * p.n;
  const uint32_t* msw = p.msw + base;
  const uint8_t* src = (f.cur ? p.loc1 : p.loc0) + base;
  uint8_t* dst = (f.cur ? p.loc0 : p.loc1) + base;
  const long long dxy = static_cast<long long>(p.dx) * p.dy;
  const long long dshift = f.off[0] + f.off[1] * static_cast<long long>(p.dx) + f.off[2] * dxy;

  unsigned occ_n = 0, free_n = 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * 4;
  for (long long c0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
       c0 < p.n; c0 += stride) {
    uint32_t out = 0;
    const int nc = p.n - c0 < 4 ? static_cast<int>(p.n - c0) : 4;
    for (int i = 0; i < nc; ++i) {
      const long long c = c0 + i;
      const int z = static_cast<int>(c / dxy);
      const long long rem = c - z * dxy;
      const int y = static_cast<int>(rem / p.dx);
      const int x = static_cast<int>(rem - static_cast<long long>(y) * p.dx);
      const int sx = x + f.off[0], sy = y + f.off[1], sz = z + f.off[2];
      uint32_t v = 0;
      if (sx >= 0 && sy >= 0 && sz >= 0 && sx < p.dx && sy < p.dy && sz < p.dz) {
        const long long sc = c + dshift;
        v = merge_cell(src[sc], decode_word(msw[sc], f.tag));
      }
      occ_n += v == 2u;
      free_n += v == 1u;
      out |= v << (8 * i);
    }
    if (nc == 4 && ((reinterpret_cast<uintptr_t>(dst + c0) & 3u) == 0)) {
      *reinterpret_cast<uint32_t*>(dst + c0) = out;
    } else {
      for (int i = 0; i < nc; ++i) dst[c0 + i] = static_cast<uint8_t>(out >> (8 * i));
    }
  }
  unsigned vals[2] = {occ_n, free_n};
  unsigned long long* dsts[2] = {&p.counters[s].occupied, &p.counters[s].freed};
  block_accumulate<2>(vals, dsts);
}

}  // namespace vxm
