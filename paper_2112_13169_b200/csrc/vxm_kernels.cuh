// The per-frame voxelization kernels (paper Alg. 1-3 + the local-grid shift).
// The last CUDA grid dimension indexes independent sensor streams, so a batch
// of S streams is one launch per stage.
//
//   K1 populate_depth / populate_cloud   depth -> point -> T_vc -> voxel -> Occupied
//   K2 dilate                           vox_inf > 0: Chebyshev dilation of the centres
//   K3 trace_bundle                     frustum ray casting, Free / UnknownTraced
//   K4 merge_shift_count                merge into the local grid, shift, count
#pragma once

#include <type_traits>

#include "vxm_device.cuh"
#include "vxm_tuning.h"

namespace vxm {

// ---------------------------------------------------------------------------
// K1: depth_to_cloud (proj/src/geometry.cpp:45-57) fused with
// voxelize_points + the centre store of mark_point (proj/src/integrator.cpp:
// 24-41, 62-85). Pixels never materialise as a point cloud;
// ((u + 0.5) - cx) / fx comes from a per-column table computed once with the
// same IEEE operations, and floor(acc / vs) avoids the fp64 division when
// provably exact (voxel_coord).
// ---------------------------------------------------------------------------
template <bool kClear>
__device__ __forceinline__ unsigned populate_point(const KParams& p, const double* R,
                                                   const double* t, uint8_t* target,
                                                   uint8_t* rowflag, uint32_t* keys, uint8_t mark, double x,
                                                   double y, double z, bool* slow = nullptr) {
  int c[3];
  transform_voxelize(R, t, x, y, z, p.vs, p.inv_vs, c, slow);
  if (static_cast<unsigned>(c[0]) >= static_cast<unsigned>(p.dx) ||
      static_cast<unsigned>(c[1]) >= static_cast<unsigned>(p.dy) ||
      static_cast<unsigned>(c[2]) >= static_cast<unsigned>(p.dz)) {
    return 1u;  // counted in points_outside
  }
  const uint32_t idx = static_cast<uint32_t>(c[0]) + static_cast<uint32_t>(c[1]) * p.dx +
                       static_cast<uint32_t>(c[2]) * (static_cast<uint32_t>(p.dx) * static_cast<uint32_t>(p.dy));
  target[idx] = mark;  // idempotent: every writer stores the same byte
  if (rowflag) {
    // a centre: the dilation only visits x-rows that hold one this frame
    rowflag[static_cast<uint32_t>(c[1]) + static_cast<uint32_t>(c[2]) * p.dy] = mark;
  } else if constexpr (kClear) {
    keys[idx] = kClearOccupied;  // vox_inf == 0: the cell itself is Occupied (clear-format keys)
  }
  return 0u;
}

// N points at once (the dense depth kernel): every point's transform and
// fast voxel coordinates first, branch-free, so that the N fp64 dependency
// chains interleave; then per valid point the bounds test and the stores of
// populate_point. Points whose floor the fast path cannot decide (rare) are
// left to the caller (bit k of *pend), so no call to the exact division sits
// in the loop (its call frame made ptxas spill the batch's registers).
template <bool kClear, int N>
__device__ __forceinline__ unsigned populate_points(const KParams& p, const double* R, const double* t,
                                                    uint8_t* target, uint8_t* rowflag, uint32_t* keys, uint8_t mark,
                                                    const double (&x)[N], const double (&y)[N], const double (&z)[N],
                                                    const bool (&ok)[N], uint32_t* pend) {
  int c[N][3];
  bool fast[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    fast[k] = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double acc = t[a];
      acc = dadd(acc, dmul(R[3 * a + 0], x[k]));
      acc = dadd(acc, dmul(R[3 * a + 1], y[k]));
      acc = dadd(acc, dmul(R[3 * a + 2], z[k]));
      bool f;
      c[k][a] = voxel_coord_fast(acc, p.vs, p.inv_vs, f);
      fast[k] = fast[k] && f;
    }
  }
  unsigned outside = 0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (!ok[k]) continue;
    if (!fast[k]) {
      *pend |= 1u << k;
      continue;
    }
    if (static_cast<unsigned>(c[k][0]) >= static_cast<unsigned>(p.dx) ||
        static_cast<unsigned>(c[k][1]) >= static_cast<unsigned>(p.dy) ||
        static_cast<unsigned>(c[k][2]) >= static_cast<unsigned>(p.dz)) {
      ++outside;
      continue;
    }
    const uint32_t idx = static_cast<uint32_t>(c[k][0]) + static_cast<uint32_t>(c[k][1]) * p.dx +
                         static_cast<uint32_t>(c[k][2]) * (static_cast<uint32_t>(p.dx) * static_cast<uint32_t>(p.dy));
    target[idx] = mark;
    if (rowflag) {
      rowflag[static_cast<uint32_t>(c[k][1]) + static_cast<uint32_t>(c[k][2]) * p.dy] = mark;
    } else if constexpr (kClear) {
      keys[idx] = kClearOccupied;
    }
  }
  return outside;
}

// Depth quads (4 pixels, one 16-byte streaming load) per thread; a block
// walks `iters` consecutive 256-quad tiles of one stream's frame and loads
// tile i+1 before resolving tile i, so the HBM latency of a batched launch
// overlaps the fp64 work.
__device__ __forceinline__ float4 load_quad(const float* depth, int first, int npix) {
  if (first + 3 < npix && (reinterpret_cast<uintptr_t>(depth + first) & 15u) == 0)
    return __ldcs(reinterpret_cast<const float4*>(depth + first));
  float d[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k] = first + k < npix ? depth[first + k] : 0.0f;
  return make_float4(d[0], d[1], d[2], d[3]);
}

template <bool kClear>
__global__ void __launch_bounds__(256) populate_depth_kernel(KParams p, int iters) {
  const int s = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_pop = global_ns();
  const FrameParams* fp = p.frames + s;
  const uint8_t mark = static_cast<uint8_t>(fp->epoch);
  uint8_t* target = (p.vox_inf > 0 ? p.ctr : p.occ) + static_cast<long long>(s) * p.n;
  uint8_t* rowflag = p.vox_inf > 0 ? p.rowflag + static_cast<long long>(s) * p.dy * p.dz : nullptr;
  uint32_t* const keys = p.key + static_cast<long long>(s) * p.n;
  double R[9], t[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = fp->rot[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = fp->trans[i];
  const float* depth = fp->depth;
  const int npix = p.W * p.H;

  unsigned total = 0, outside = 0;
  float mind = __uint_as_float(0x7F800000u);
  int first = ((blockIdx.x * iters) * blockDim.x + threadIdx.x) * 4;
  float4 next = first < npix ? load_quad(depth, first, npix) : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int it = 0; it < iters && first < npix; ++it) {
    const float4 cur = next;
    const int nfirst = first + blockDim.x * 4;
    if (it + 1 < iters && nfirst < npix) next = load_quad(depth, nfirst, npix);
    const float d[4] = {cur.x, cur.y, cur.z, cur.w};
    const int v0 = first / p.W;
    const int u0 = first - v0 * p.W;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int u = u0 + k, v = v0;
      if (u >= p.W) { u -= p.W; ++v; }  // a row boundary inside the quad
      // DepthImage::valid_depth (geometry.hpp:124): finite and > 0; then the
      // max-depth cut on the promoted double (geometry.cpp:53-54).
      if (first + k >= npix || !(isfinite(d[k]) && d[k] > 0.0f)) continue;
      const double D = static_cast<double>(d[k]);
      if (D > p.max_depth) continue;
      ++total;
      mind = fminf(mind, d[k]);  // |point| >= its depth
      outside += populate_point<kClear>(p, R, t, target, rowflag, keys, mark, dmul(__ldg(p.qx + u), D),
                                dmul(__ldg(p.qy + v), D), D);
    }
    first = nfirst;
  }
  warp_min_dist(mind, &p.counters[s].min_dist_bits);
  unsigned vals[2] = {total, outside};
  unsigned long long* dst[2] = {&p.counters[s].points_total, &p.counters[s].points_outside};
  block_accumulate<2>(vals, dst);
}

// K1 with the depth span of a block staged in shared memory by the TMA
// engine: one elected thread issues `iters` bulk copies (one per 256-quad
// tile, 4 KB each) on per-tile mbarriers at block start, so every block keeps
// its whole span in flight (HBM latency no longer bounds the launch); the
// threads then consume tile after tile as the copies land. kCompact: each
// warp first lists its valid pixels and transforms them densely (frames with
// many invalid / out-of-range pixels); the host picks the variant from the
// valid fraction it last observed. Requires W*H % 4 == 0 and a 16-byte
// aligned frame (checked; otherwise the plain loads).
constexpr int kPopMaxIters = 8;

template <bool kCompact, bool kClear>
__global__ void __launch_bounds__(256, VXM_POP_MINB) populate_depth_tma_kernel(KParams p, int iters) {
  extern __shared__ float4 sq[];  // iters * blockDim.x quads
  __shared__ uint64_t bar[kPopMaxIters];
  const int s = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_pop = global_ns();
  const FrameParams* fp = p.frames + s;
  const uint8_t mark = static_cast<uint8_t>(fp->epoch);
  uint8_t* target = (p.vox_inf > 0 ? p.ctr : p.occ) + static_cast<long long>(s) * p.n;
  uint8_t* rowflag = p.vox_inf > 0 ? p.rowflag + static_cast<long long>(s) * p.dy * p.dz : nullptr;
  uint32_t* const keys = p.key + static_cast<long long>(s) * p.n;
  const float* depth = fp->depth;
  const int nq = (p.W * p.H) >> 2;
  const int T = blockDim.x;
  const int q0 = blockIdx.x * iters * T;
  const bool aligned = (reinterpret_cast<uintptr_t>(depth) & 15u) == 0;
  if (aligned && threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    for (int i = 0; i < iters; ++i) {
      const int start = q0 + i * T;
      if (start >= nq) break;
      const uint32_t bytes = static_cast<uint32_t>(min(T, nq - start)) * 16u;
      mbar_expect_tx(&bar[i], bytes);
#if VXM_POP_EVICT_FIRST
      bulk_g2s_stream(sq + i * T, depth + static_cast<long long>(start) * 4, bytes, &bar[i]);
#else
      bulk_g2s(sq + i * T, depth + static_cast<long long>(start) * 4, bytes, &bar[i]);
#endif
    }
  }
  double R[9], t[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = fp->rot[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = fp->trans[i];
  __syncthreads();  // barriers initialised before anyone waits on them

  unsigned total = 0, outside = 0;
  float mind = __uint_as_float(0x7F800000u);
  if constexpr (kCompact) {
  // Each warp lists the valid pixels of its own quads (ballot positions, no
  // block barrier) and then transforms them 32 at a time, so no lane idles on
  // an invalid pixel (sparse frames: a cfg2 frame is ~70% beyond max_depth).
  uint16_t* wl = reinterpret_cast<uint16_t*>(sq + iters * T) + (threadIdx.x >> 5) * (iters * 128);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int nlist = 0;
  for (int it = 0; it < iters; ++it) {
    if (q0 + it * T >= nq) break;
    const int q = q0 + it * T + threadIdx.x;
    float4 cur = make_float4(0.f, 0.f, 0.f, 0.f);
    if (aligned) {
      mbar_wait(&bar[it], 0);
      if (q < nq) cur = sq[it * T + threadIdx.x];
    } else if (q < nq) {
      cur = load_quad(depth, q * 4, nq * 4);
      sq[it * T + threadIdx.x] = cur;
    }
    const float d[4] = {cur.x, cur.y, cur.z, cur.w};
    bool ok[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // DepthImage::valid_depth (geometry.hpp:124): finite and > 0; then the
      // max-depth cut on the promoted double (geometry.cpp:53-54). With
      // max_depth_f the largest float <= max_depth, "d > 0 && d <= max_depth_f"
      // is the same test (NaN and +inf fail the second compare).
      ok[k] = q < nq && d[k] > 0.0f && d[k] <= p.max_depth_f;
    }
    // most 128-pixel groups of a sparse frame hold no valid pixel
    if (__any_sync(0xffffffffu, ok[0] || ok[1] || ok[2] || ok[3])) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned b = __ballot_sync(0xffffffffu, ok[k]);
        if (ok[k]) wl[nlist + __popc(b & lt)] = static_cast<uint16_t>((it * T + threadIdx.x) * 4 + k);
        nlist += __popc(b);
      }
    }
  }
  __syncwarp();
  const float* spx = reinterpret_cast<const float*>(sq);
  const int pix0 = q0 * 4;
  const float invW = 1.0f / static_cast<float>(p.W);
  total += lane == 0 ? static_cast<unsigned>(nlist) : 0u;
  auto pixel_uv = [&](int off, int& u, int& v) {
    const int pix = pix0 + off;
    v = static_cast<int>((static_cast<float>(pix) + 0.5f) * invW);  // pix / W, corrected below
    v -= v * p.W > pix ? 1 : 0;
    v += (v + 1) * p.W <= pix ? 1 : 0;
    u = pix - v * p.W;
  };
#if VXM_POP_CBATCH
  // VXM_POP_CBATCH list entries per lane at a time (interleaved fp64 chains);
  // entry 32 j + lane whose floor the fast path cannot decide sets bit j of
  // `pending` (a warp lists at most iters * 128 <= 1024 pixels, so j < 32)
  constexpr int B = VXM_POP_CBATCH;
  uint32_t pending = 0;
  int i0 = 0;
  for (; i0 < nlist; i0 += 32 * B) {
    double X[B], Y[B], Z[B];
    bool ok[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int i = i0 + 32 * b + lane;
      ok[b] = i < nlist;
      const int off = ok[b] ? wl[i] : 0;
      int u, v;
      pixel_uv(off, u, v);
      const float dk = spx[off];
      const double D = static_cast<double>(ok[b] ? dk : 0.0f);
      mind = ok[b] ? fminf(mind, dk) : mind;
      X[b] = dmul(__ldg(p.qx + u), D);
      Y[b] = dmul(__ldg(p.qy + v), D);
      Z[b] = D;
    }
    uint32_t pm = 0;
    outside += populate_points<kClear, B>(p, R, t, target, rowflag, keys, mark, X, Y, Z, ok, &pm);
    pending |= pm << (i0 >> 5);
    // many deferred points (voxel faces): the rest one at a time, as the dense path
    if (__popc(__ballot_sync(0xffffffffu, pm != 0u)) > VXM_POP_SERIAL_LANES) {
      i0 += 32 * B;
      break;
    }
  }
  for (int i = i0 + lane; i < nlist; i += 32) {
    const int off = wl[i];
    int u, v;
    pixel_uv(off, u, v);
    const double D = static_cast<double>(spx[off]);
    mind = fminf(mind, spx[off]);
    outside += populate_point<kClear>(p, R, t, target, rowflag, keys, mark, dmul(__ldg(p.qx + u), D),
                              dmul(__ldg(p.qy + v), D), D);
  }
  while (pending) {
    const int j = __ffs(pending) - 1;
    pending &= pending - 1;
    const int off = wl[32 * j + lane];
    int u, v;
    pixel_uv(off, u, v);
    const double D = static_cast<double>(spx[off]);
    outside += populate_point<kClear>(p, R, t, target, rowflag, keys, mark, dmul(__ldg(p.qx + u), D),
                              dmul(__ldg(p.qy + v), D), D);
  }
#else
  for (int i = lane; i < nlist; i += 32) {
    const int off = wl[i];
    int u, v;
    pixel_uv(off, u, v);
    const double D = static_cast<double>(spx[off]);
    mind = fminf(mind, spx[off]);
    outside += populate_point<kClear>(p, R, t, target, rowflag, keys, mark, dmul(__ldg(p.qx + u), D),
                              dmul(__ldg(p.qy + v), D), D);
  }
#endif
  } else {
  // the thread's first pixel (u0, v0) advances by 4T pixels per tile: one
  // division for the first tile, then a carry
  int v0 = (q0 * 4 + threadIdx.x * 4) / p.W;
  int u0 = q0 * 4 + threadIdx.x * 4 - v0 * p.W;
  const int du = (4 * T) % p.W, dv = (4 * T) / p.W;
  uint32_t pending = 0;  // bit 4 it + k: pixel k of tile it needs the exact division (iters <= 8)
  // (warp-uniform) the rest of the tiles one pixel at a time: from the start
  // when most warps of the slot's previous K1 found face-heavy tiles
  const uint32_t hint = __ldcg(&p.counters[s].pop_faces) >> 16;
  bool serial = 100u * hint > VXM_POP_HINT_PCT * gridDim.x * (blockDim.x >> 5);
  bool faces = false;  // this warp's first tile was face-heavy
  bool lane_slow = false;  // (serial, first tile) a pixel of this lane took the slow floor
  for (int it = 0; it < iters; ++it, u0 += du, v0 += dv) {
    if (u0 >= p.W) { u0 -= p.W; ++v0; }
    const int q = q0 + it * T + threadIdx.x;
    if (q0 + it * T >= nq) break;
    float4 cur;
    if (aligned) {
      mbar_wait(&bar[it], 0);
      cur = q < nq ? sq[it * T + threadIdx.x] : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      cur = q < nq ? load_quad(depth, q * 4, nq * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (q >= nq) continue;
    const float d[4] = {cur.x, cur.y, cur.z, cur.w};
#if VXM_POP_BATCH
    if (!serial) {
    double X[4], Y[4], Z[4];
    bool ok[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int u = u0 + k, v = v0;
      if (u >= p.W) { u -= p.W; ++v; }  // a row boundary inside the quad
      // DepthImage::valid_depth (geometry.hpp:124): finite and > 0; then the
      // max-depth cut on the promoted double (geometry.cpp:53-54), as two
      // float compares against the largest float <= max_depth
      ok[k] = d[k] > 0.0f && d[k] <= p.max_depth_f;
      const double D = static_cast<double>(ok[k] ? d[k] : 0.0f);
      total += ok[k] ? 1u : 0u;
      mind = ok[k] ? fminf(mind, d[k]) : mind;
      X[k] = dmul(__ldg(p.qx + u), D);
      Y[k] = dmul(__ldg(p.qy + v), D);
      Z[k] = D;
    }
#pragma unroll
    for (int h = 0; h < 4; h += VXM_POP_BATCH) {
      double x[VXM_POP_BATCH], y[VXM_POP_BATCH], z[VXM_POP_BATCH];
      bool o[VXM_POP_BATCH];
#pragma unroll
      for (int k = 0; k < VXM_POP_BATCH; ++k) {
        x[k] = X[h + k];
        y[k] = Y[h + k];
        z[k] = Z[h + k];
        o[k] = ok[h + k];
      }
      uint32_t pm = 0;
      outside += populate_points<kClear, VXM_POP_BATCH>(p, R, t, target, rowflag, keys, mark, x, y, z, o, &pm);
      pending |= pm << (4 * it + h);
    }
    // Points on voxel faces (axis-aligned walls and floors, e.g. a corridor)
    // are deferred almost all: a warp whose tile deferred pixels on more than
    // VXM_POP_SERIAL_LANES lanes takes the rest of its tiles one pixel at a
    // time with the near-integer floor inline (populate_point), which costs
    // less there than the batch plus the deferred pass.
    serial = __popc(__ballot_sync(__activemask(), ((pending >> (4 * it)) & 0xFu) != 0u)) > VXM_POP_SERIAL_LANES;
    faces = faces || (it == 0 && serial);
    continue;
    }
#endif
    {
    bool* slow = it == 0 ? &lane_slow : nullptr;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int u = u0 + k, v = v0;
      if (u >= p.W) { u -= p.W; ++v; }  // a row boundary inside the quad
      // DepthImage::valid_depth (geometry.hpp:124): finite and > 0; then the
      // max-depth cut on the promoted double (geometry.cpp:53-54), as two
      // float compares against the largest float <= max_depth
      if (!(d[k] > 0.0f && d[k] <= p.max_depth_f)) continue;
      const double D = static_cast<double>(d[k]);
      ++total;
      mind = fminf(mind, d[k]);
      outside += populate_point<kClear>(p, R, t, target, rowflag, keys, mark, dmul(__ldg(p.qx + u), D),
                                dmul(__ldg(p.qy + v), D), D, slow);
    }
    if (it == 0) faces = __popc(__ballot_sync(__activemask(), lane_slow)) > VXM_POP_SERIAL_LANES;
    }
  }
  if (faces && (threadIdx.x & 31) == 0) atomicAdd(&p.counters[s].pop_faces, 1u);
  // the pixels the fast floor could not decide, through populate_point (the
  // exact division); the depth is still in shared memory (or re-read)
  while (pending) {
    const int b = __ffs(pending) - 1;
    pending &= pending - 1;
    const int it = b >> 2, k = b & 3;
    const int q = q0 + it * T + threadIdx.x;
    const float dk = aligned ? reinterpret_cast<const float*>(sq + it * T + threadIdx.x)[k] : depth[q * 4 + k];
    const int pix = q * 4 + k;
    const int v = pix / p.W, u = pix - v * p.W;
    const double D = static_cast<double>(dk);
    outside += populate_point<kClear>(p, R, t, target, rowflag, keys, mark, dmul(__ldg(p.qx + u), D),
                              dmul(__ldg(p.qy + v), D), D);
  }
  }
  warp_min_dist(mind, &p.counters[s].min_dist_bits);
  unsigned vals[2] = {total, outside};
  unsigned long long* dst[2] = {&p.counters[s].points_total, &p.counters[s].points_outside};
  warp_accumulate<2>(vals, dst);
}

// K1 for an explicit camera-frame cloud (MeasurementFrame::cloud). Points
// that PointCloud::add would have dropped (non-finite) are skipped uncounted
// (proj/include/voxmap/geometry.hpp:84-89).
template <bool kClear>
__global__ void __launch_bounds__(256) populate_cloud_kernel(KParams p) {
  const int s = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_pop = global_ns();
  const FrameParams* fp = p.frames + s;
  const uint8_t mark = static_cast<uint8_t>(fp->epoch);
  uint8_t* target = (p.vox_inf > 0 ? p.ctr : p.occ) + static_cast<long long>(s) * p.n;
  uint8_t* rowflag = p.vox_inf > 0 ? p.rowflag + static_cast<long long>(s) * p.dy * p.dz : nullptr;
  uint32_t* const keys = p.key + static_cast<long long>(s) * p.n;
  double R[9], t[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = fp->rot[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = fp->trans[i];
  const long long n = fp->n_points;
  const double *xs = fp->xs, *ys = fp->ys, *zs = fp->zs;
  unsigned total = 0, outside = 0;
  float mind = __uint_as_float(0x7F800000u);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double x = xs[i], y = ys[i], z = zs[i];
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) continue;
    ++total;
    // a lower bound of |point|, rounded down to a float
    mind = fminf(mind, __double2float_rd(fmax(fabs(x), fmax(fabs(y), fabs(z)))));
    outside += populate_point<kClear>(p, R, t, target, rowflag, keys, mark, x, y, z);
  }
  warp_min_dist(mind, &p.counters[s].min_dist_bits);
  unsigned vals[2] = {total, outside};
  unsigned long long* dst[2] = {&p.counters[s].points_total, &p.counters[s].points_outside};
  block_accumulate<2>(vals, dst);
}

// ---------------------------------------------------------------------------
// K2: obstacle inflation. mark_point writes the (2r+1)^3 cube around every
// in-bounds centre, clipped to the grid (integrator.cpp:70-83): a Chebyshev
// dilation of the centre set restricted to the grid, which is separable.
// Two kernels: K2a packs and x-dilates every row once into a bit plane; K2b
// dilates 8x8 tiles of bit rows along y and z in shared memory and writes the
// Occupied bytes.
// ---------------------------------------------------------------------------
// (y, z) tile edge of the dilation (a power of two): 8 for batches, 4 for a
// lone frame (more blocks for one frame: 30.7 -> 28.7 us per cfg2 frame; 16
// and 4 measured slower for 64-stream batches, profiles/r02ad_dil_tile_ab.txt)
constexpr int kDilT = 8;
constexpr int kDilTLone = 4;

// Word stride of a bit row: ceil(dx/32) rounded up to a power of two, so the
// index arithmetic is shifts and masks.
__host__ __device__ constexpr int dilate_row_words(int dx) {
  int w = 1;
  while (w * 32 < dx) w <<= 1;
  return w;
}

// K2a: one warp per x-row: the row's centre bytes become a bit row (one
// ballot per 32 cells, coalesced byte loads), dilated along x by r with
// shuffles between the lanes holding neighbouring words, and stored to the
// per-stream bit plane `dbits` [dy*dz rows][WP words]. Each row is packed
// exactly once (the tile kernel below reads bits, never bytes).
constexpr int kDilRowsPerWarp = 4;

__global__ void __launch_bounds__(256) dilate_rows_kernel(KParams p, int r) {
  pdl_wait();  // K1's centre bytes and row flags
  const int s = blockIdx.y;
  const uint32_t e = p.frames[s].epoch;
  const int lane = threadIdx.x & 31;
  const int row0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kDilRowsPerWarp;
  const int rows = p.dy * p.dz;
  const int W = (p.dx + 31) >> 5;
  const int WP = dilate_row_words(p.dx);
  const uint8_t* ctr = p.ctr + static_cast<long long>(s) * p.n;
  uint32_t* plane = p.dbits + static_cast<long long>(s) * rows * WP;
  const uint8_t* rf = p.rowflag + static_cast<long long>(s) * rows;
  for (int row = row0; row < row0 + kDilRowsPerWarp && row < rows; ++row) {
    if (rf[row] != e) continue;  // no centre in this row (K2b never reads its bits)
    const uint8_t* src = ctr + static_cast<uint32_t>(row) * p.dx;
    uint32_t mine = 0;  // lane w keeps word w
    for (int w0 = 0; w0 < W; w0 += 4) {
      uint32_t c[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int x = ((w0 + j) << 5) + lane;
        c[j] = x < p.dx ? __ldg(src + x) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t m = __ballot_sync(0xffffffffu, c[j] == e);
        if (lane == w0 + j) mine = m;
      }
    }
    uint32_t d = mine;
    if (__any_sync(0xffffffffu, mine != 0u)) {
      const uint32_t prev = __shfl_up_sync(0xffffffffu, mine, 1);
      const uint32_t next = __shfl_down_sync(0xffffffffu, mine, 1);
      const uint32_t pv = lane > 0 ? prev : 0u;
      const uint32_t nx = lane + 1 < W ? next : 0u;
      for (int k = 1; k <= r; ++k) d |= (mine << k) | (pv >> (32 - k)) | (mine >> k) | (nx << (32 - k));
    }
    if (lane < WP) plane[static_cast<uint32_t>(row) * WP + lane] = lane < W ? d : 0u;
  }
}

// K2a, vector form: a warp packs a group of G consecutive rows whose bytes
// (G*dx) form whole 16-byte vectors (one 16-byte streaming load per lane,
// G*dx <= 512). Each lane turns its 16 bytes into a 16-bit mask; lane o < G*WP
// then assembles word (o & (WP-1)) of row (o / WP) from the masks of the
// (at most) three lanes covering it, clears the bits past dx, dilates along x
// with its neighbouring words, and stores it. Used when the stream size and
// G*dx are multiples of 16 (all benchmark grids); else the per-row kernel.
__host__ __device__ constexpr int dilate_rows_group(int dx) {
  // smallest G with G*dx % 16 == 0 (1, 2, 4, 8, 16)
  int g = 1;
  while ((g * dx) % 16 != 0) g <<= 1;
  return g;
}

__global__ void __launch_bounds__(256) dilate_rows_vec_kernel(KParams p, int r) {
  pdl_wait();  // K1's centre bytes and row flags
  const int s = blockIdx.y;
  const uint32_t e = p.frames[s].epoch;
  const int lane = threadIdx.x & 31;
  const int G = dilate_rows_group(p.dx);
  const int WP = dilate_row_words(p.dx);
  const int lg = __ffs(WP) - 1;
  const int W = (p.dx + 31) >> 5;
  const int rows = p.dy * p.dz;
  const int row0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G;
  if (row0 >= rows) return;
  // rows without a centre this frame are skipped (K2b never reads their bits)
  const uint8_t* rf = p.rowflag + static_cast<long long>(s) * rows;
  if (!__any_sync(0xffffffffu, lane < G && row0 + lane < rows && rf[row0 + lane] == e)) return;
  const int span = min(G, rows - row0) * p.dx;  // bytes of this group
  const uint8_t* src = p.ctr + static_cast<long long>(s) * p.n + static_cast<long long>(row0) * p.dx;
  uint32_t m = 0;  // bit i: byte 16*lane + i holds a centre
  if (lane * 16 < span) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src) + lane);
    const uint32_t ee = e * 0x01010101u;
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t hit = zero_bytes_msb(w4[i] ^ ee);  // 0x80 per matching byte
      m |= ((hit * 0x00204081u) >> 28) << (4 * i);
    }
  }
  // word j of row k covers group bytes [k*dx + 32j, +32)
  const int k = lane >> lg, j = lane & (WP - 1);
  const int b0 = k * p.dx + 32 * j;
  const int L0 = b0 >> 4, off = b0 & 15;
  const uint32_t m0 = __shfl_sync(0xffffffffu, m, L0 & 31);
  const uint32_t m1 = __shfl_sync(0xffffffffu, m, (L0 + 1) & 31);
  const uint32_t m2 = __shfl_sync(0xffffffffu, m, (L0 + 2) & 31);
  const unsigned long long win = static_cast<unsigned long long>(m0) | (static_cast<unsigned long long>(m1) << 16) |
                                 (static_cast<unsigned long long>(m2) << 32);
  const int valid = min(32, p.dx - 32 * j);  // cells of this word inside the row
  uint32_t w = j < W ? static_cast<uint32_t>(win >> off) : 0u;
  if (valid < 32) w &= valid > 0 ? (1u << valid) - 1u : 0u;
  uint32_t d = w;
  if (__any_sync(0xffffffffu, w != 0u)) {
    const uint32_t prev = __shfl_up_sync(0xffffffffu, w, 1);
    const uint32_t next = __shfl_down_sync(0xffffffffu, w, 1);
    const uint32_t pv = j > 0 ? prev : 0u;
    const uint32_t nx = j + 1 < WP ? next : 0u;
    for (int q = 1; q <= r; ++q) d |= (w << q) | (pv >> (32 - q)) | (w >> q) | (nx << (32 - q));
    if (valid < 32) d &= valid > 0 ? (1u << valid) - 1u : 0u;
  }
  if (k < G && row0 + k < rows) {
    uint32_t* plane = p.dbits + static_cast<long long>(s) * rows * WP;
    plane[static_cast<uint32_t>(row0 + k) * WP + j] = d;
  }
}

// Shared memory of K2b: the (8+2r)^2 halo bit rows and the y-dilated rows
// (fused: also the packed, not yet x-dilated, halo rows).
__host__ __device__ constexpr size_t dilate_smem_bytes(int r, int dx, bool fused = false, int T = kDilT) {
  return sizeof(uint32_t) * static_cast<size_t>(dilate_row_words(dx)) *
             (static_cast<size_t>(T + 2 * r) * (T + 2 * r) * (fused ? 2 : 1) +
              static_cast<size_t>(T) * (T + 2 * r)) +
         ((static_cast<size_t>(T + 2 * r) * (T + 2 * r) + 3) & ~static_cast<size_t>(3));  // row flags
}

// K2b: a block owns an 8x8 (y,z) tile of x-dilated bit rows, loads them with
// an r-row halo into shared memory, ORs along y then z, and writes one
// Occupied byte per set bit (a warp covers 32 consecutive cells).
// kR > 0: radius fixed at compile time; kR == 0: radius at run time.
// kFused: no K2a; the block packs and x-dilates its halo rows itself from the
// centre bytes (dims_x % 4 == 0: 4-byte loads), one launch fewer.
template <int kR, bool kFused, bool kClear, int kT = kDilT>
__global__ void __launch_bounds__(256) dilate_tiles_kernel(KParams p, int r_rt) {
  pdl_wait();  // K1's centre bytes (fused) or K2a's bit rows
  extern __shared__ uint32_t bits[];
  const int r = kR > 0 ? kR : r_rt;
  const int s = blockIdx.z;
  const uint32_t e = p.frames[s].epoch;
  uint8_t* occ = p.occ + static_cast<long long>(s) * p.n;
  uint32_t* const keys = p.key + static_cast<long long>(s) * p.n;
  const int W = (p.dx + 31) >> 5;
  const int WP = dilate_row_words(p.dx);
  const int lg = __ffs(WP) - 1;
  const int H = kT + 2 * r;
  const int y0 = blockIdx.x * kT, z0 = blockIdx.y * kT;
  const uint32_t dxy = static_cast<uint32_t>(p.dx) * p.dy;
  const uint32_t* plane = p.dbits + static_cast<long long>(s) * p.dy * p.dz * WP;
  uint32_t* bx = bits;                  // [H z][H y][WP]
  uint32_t* by = bx + (H * H << lg);    // [H z][kT y][WP], y-dilated
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;

  uint8_t* fl = reinterpret_cast<uint8_t*>(by + ((H * kT) << lg));  // [H z][H y] row holds a centre
  const uint8_t* rf = p.rowflag + static_cast<long long>(s) * p.dy * p.dz;
  bool anyf = false;
  for (int i = threadIdx.x; i < H * H; i += blockDim.x) {
    const int hz = i / H, hy = i - hz * H;
    const int y = y0 - r + hy, z = z0 - r + hz;
    const bool f = y >= 0 && y < p.dy && z >= 0 && z < p.dz &&
                   rf[static_cast<uint32_t>(z) * static_cast<uint32_t>(p.dy) + static_cast<uint32_t>(y)] == e;
    fl[i] = f ? 1 : 0;
    anyf = anyf || f;
  }
  // surfaces are sparse in 3-D: a tile with no centre within r writes nothing
  if (!__syncthreads_or(anyf)) return;
  if constexpr (kFused) {
    // pack: word w of a flagged halo row = its 32 centre bytes == epoch
    uint32_t* raw = reinterpret_cast<uint32_t*>(fl + ((H * H + 3) & ~3)) ;
    const uint8_t* ctr = p.ctr + static_cast<long long>(s) * p.n;
    const uint32_t ee = e * 0x01010101u;
    for (int i = threadIdx.x; i < (H * H) << lg; i += blockDim.x) {
      const int w = i & (WP - 1), row = i >> lg;
      uint32_t m = 0;
      if (fl[row] && w < W) {
        const int hz = row / H, hy = row - hz * H;
        const int y = y0 - r + hy, z = z0 - r + hz;
        const uint32_t* src =
            reinterpret_cast<const uint32_t*>(ctr + static_cast<uint32_t>(y) * p.dx + static_cast<uint32_t>(z) * dxy) +
            8 * w;
        const int nq = min(8, (p.dx - 32 * w) >> 2);  // 4-byte words of this 32-cell word inside the row
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < nq) {
            const uint32_t hit = zero_bytes_msb(__ldg(src + q) ^ ee);  // 0x80 per centre byte
            m |= ((hit * 0x00204081u) >> 28) << (4 * q);
          }
        }
      }
      raw[i] = m;
    }
    __syncthreads();
    // x-dilation with the neighbouring words of the row
    for (int i = threadIdx.x; i < (H * H) << lg; i += blockDim.x) {
      const int w = i & (WP - 1);
      const uint32_t m = raw[i];
      const uint32_t pv = w > 0 ? raw[i - 1] : 0u;
      const uint32_t nx = w + 1 < W ? raw[i + 1] : 0u;
      uint32_t d = m;
      if (m | pv | nx) {
#pragma unroll
        for (int q = 1; q <= (kR > 0 ? kR : 16); ++q) {
          if (kR == 0 && q > r) break;
          d |= (m << q) | (pv >> (32 - q)) | (m >> q) | (nx << (32 - q));
        }
        const int valid = min(32, p.dx - 32 * w);
        if (valid < 32) d &= valid > 0 ? (1u << valid) - 1u : 0u;
      }
      bx[i] = w < W ? d : 0u;
    }
  } else {
    for (int i = threadIdx.x; i < (H * H) << lg; i += blockDim.x) {
      const int w = i & (WP - 1), row = i >> lg;
      const int hz = row / H, hy = row - hz * H;
      const int y = y0 - r + hy, z = z0 - r + hz;
      bx[i] = fl[row] ? __ldg(plane + ((static_cast<long long>(z) * p.dy + y) << lg) + w) : 0u;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (H * kT) << lg; i += blockDim.x) {
    const int w = i & (WP - 1), yz = i >> lg;
    const int y = yz & (kT - 1), hz = yz / kT;
    const uint32_t* col = bx + ((hz * H + y) << lg) + w;
    uint32_t d = 0;
#pragma unroll
    for (int k = 0; k <= 2 * (kR > 0 ? kR : 16); ++k) {
      if (kR == 0 && k > 2 * r) break;
      d |= col[k << lg];
    }
    by[i] = d;
  }
  __syncthreads();
  if (!kClear && nw == kT && (p.dx & 3) == 0 && p.dx <= 128) {
    // one warp per y row of the tile (8 warps, 8x8 tile), walking its z
    // column with running pointers; a lane owns one 4-cell group of the row
    const int gy = y0 + warp, x0 = lane * 4;
    if (gy < p.dy && x0 < p.dx) {
      const int zs = kT << lg;
      const uint32_t* col = by + (warp << lg) + (x0 >> 5);
      uint8_t* dst = occ + static_cast<uint32_t>(gy) * p.dx + static_cast<uint32_t>(z0) * dxy + x0;
      const int zn = min(kT, p.dz - z0);
      const uint32_t ee = e * 0x01010101u;
      for (int z = 0; z < zn; ++z, col += zs, dst += dxy) {
        uint32_t d = 0;
#pragma unroll
        for (int k = 0; k <= 2 * (kR > 0 ? kR : 16); ++k) {
          if (kR == 0 && k > 2 * r) break;
          d |= col[k * zs];
        }
        const uint32_t nib = (d >> (x0 & 31)) & 0xFu;
        if (nib) *reinterpret_cast<uint32_t*>(dst) = ee & (((nib * 0x00204081u) & 0x01010101u) * 0xFFu);
      }
    }
    return;
  }
  for (int row = warp; row < kT * kT; row += nw) {
    const int z = row / kT, y = row & (kT - 1);
    const int gy = y0 + y, gz = z0 + z;
    if (gy >= p.dy || gz >= p.dz) continue;
    uint8_t* dst = occ + static_cast<uint32_t>(gy) * p.dx + static_cast<uint32_t>(gz) * dxy;
    if ((p.dx & 3) == 0) {
      // 4 cells per lane, one 32-bit store per word holding a dilated cell:
      // the tile owns its rows and the only other bytes this frame could
      // have set are its own, so the rest of the word may become 0 (never an
      // epoch); the stage API restores pre-existing Occupied cells itself
      for (int x0 = lane * 4; x0 < p.dx; x0 += 128) {
        const uint32_t* col = by + ((z * kT + y) << lg) + (x0 >> 5);
        uint32_t d = 0;
#pragma unroll
        for (int k = 0; k <= 2 * (kR > 0 ? kR : 16); ++k) {
          if (kR == 0 && k > 2 * r) break;
          d |= col[(k * kT) << lg];
        }
        const uint32_t nib = (d >> (x0 & 31)) & 0xFu;
        if (nib) {
          const uint32_t m = ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;  // 0xFF per set bit
          *reinterpret_cast<uint32_t*>(dst + x0) = e * 0x01010101u & m;
          // clear-format keys: Occupied where set, Unknown (as every key is
          // before the trace) elsewhere
          if constexpr (kClear) {
            const uint32_t cell = static_cast<uint32_t>(gy) * p.dx + static_cast<uint32_t>(gz) * dxy + x0;
            *reinterpret_cast<uint4*>(keys + cell) =
                make_uint4(0u - (nib & 1u), 0u - ((nib >> 1) & 1u), 0u - ((nib >> 2) & 1u), 0u - (nib >> 3));
          }
        }
      }
      continue;
    }
    for (int w = 0; w < W; ++w) {
      const uint32_t* col = by + ((z * kT + y) << lg) + w;
      uint32_t d = 0;
#pragma unroll
      for (int k = 0; k <= 2 * (kR > 0 ? kR : 16); ++k) {
        if (kR == 0 && k > 2 * r) break;
        d |= col[(k * kT) << lg];
      }
      const int x = (w << 5) + lane;
      if (x < p.dx && ((d >> lane) & 1u)) {
        dst[x] = static_cast<uint8_t>(e);
        if constexpr (kClear) keys[static_cast<uint32_t>(gy) * p.dx + static_cast<uint32_t>(gz) * dxy + x] = kClearOccupied;
      }
    }
  }
}

// Generic K2 for what the tile kernels do not cover (vox_inf > kMaxVoxInf,
// rows longer than 1024 cells, or tiles whose shared memory would not fit):
// the same separable Chebyshev dilation as three line passes with a running
// window count (any radius, O(N) per pass): x over the centre bytes (== e)
// into tmp0, y over tmp0 into tmp1, z over tmp1 into the Occupied bytes and
// keys. Lines along y and z map consecutive threads to consecutive x
// (coalesced); lines along x are one row per thread.
__global__ void __launch_bounds__(256) dilate_line_kernel(KParams p, int r, int axis) {
  pdl_wait();  // K1's centre bytes (axis 0) or the previous pass
  const int s = blockIdx.y;
  const uint32_t e = p.frames[s].epoch;
  const long long n = p.n;
  const long long dx = p.dx, dy = p.dy, dz = p.dz, dxy = dx * dy;
  uint8_t* const t0 = p.dtmp + static_cast<long long>(s) * 2 * n;
  uint8_t* const t1 = t0 + n;
  const uint8_t* in = axis == 0 ? p.ctr + static_cast<long long>(s) * n : (axis == 1 ? t0 : t1);
  uint8_t* out = axis == 0 ? t0 : t1;
  uint8_t* occ = p.occ + static_cast<long long>(s) * n;
  uint32_t* const keys = p.key + static_cast<long long>(s) * p.n;
  const long long len = axis == 0 ? dx : (axis == 1 ? dy : dz);
  const long long stride = axis == 0 ? 1 : (axis == 1 ? dx : dxy);
  const long long lines = n / len;
  for (long long L = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; L < lines;
       L += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long base;
    if (axis == 0) base = L * dx;                                   // row (y, z)
    else if (axis == 1) base = (L % dx) + (L / dx) * dxy;           // column (x, z)
    else base = L;                                                  // pillar (x, y)
    auto set = [&](long long i) -> int {
      const uint8_t v = in[base + i * stride];
      return axis == 0 ? (v == e) : (v != 0);
    };
    int cnt = 0;  // set cells in [i - r, i + r] of the line
    for (long long j = 0; j <= r && j < len; ++j) cnt += set(j);
    for (long long i = 0; i < len; ++i) {
      const long long c = base + i * stride;
      if (axis < 2) {
        out[c] = cnt > 0 ? 1 : 0;
      } else if (cnt > 0) {
        occ[c] = static_cast<uint8_t>(e);
        store_occupied_key(keys, static_cast<uint32_t>(c), p.key_fmt);
      }
      if (i + r + 1 < len) cnt += set(i + r + 1);
      if (i - r >= 0) cnt -= set(i - r);
    }
  }
}

inline bool dilate_generic(int r, int dx);

// Launches K2a and the radius-specialised K2b (1..4) or the generic one.
// The fused K2 (no K2a) when the centre rows load as 4-byte words and its
// shared memory fits.
inline bool dilate_fused(int r, int dx) {
  return dx % 4 == 0 && dilate_smem_bytes(r, dx, true) <= 200 * 1024;
}

template <int kR, bool kClear, int kT>
inline void launch_dilate_tiles_k(const KParams& kp, int r, bool fused, cudaStream_t st, int streams) {
  const dim3 grid((kp.dy + kT - 1) / kT, (kp.dz + kT - 1) / kT, streams);
  if (fused)
    launch_pdl(dilate_tiles_kernel<kR, true, kClear, kT>, grid, dim3(256), dilate_smem_bytes(r, kp.dx, true, kT), st,
               kp, r);
  else
    launch_pdl(dilate_tiles_kernel<kR, false, kClear, kT>, grid, dim3(256), dilate_smem_bytes(r, kp.dx, false, kT),
               st, kp, r);
}
template <int kR>
inline void launch_dilate_tiles(const KParams& kp, int r, bool fused, cudaStream_t st, int streams) {
  const bool lone = streams <= 2;
  if (kp.key_fmt == kClearKeys) {
    if (lone) launch_dilate_tiles_k<kR, true, kDilTLone>(kp, r, fused, st, streams);
    else launch_dilate_tiles_k<kR, true, kDilT>(kp, r, fused, st, streams);
  } else {
    if (lone) launch_dilate_tiles_k<kR, false, kDilTLone>(kp, r, fused, st, streams);
    else launch_dilate_tiles_k<kR, false, kDilT>(kp, r, fused, st, streams);
  }
}

// the tile dilation's limits (radius, row length, shared memory)
inline bool dilate_generic(int r, int dx) {
  return r > kMaxVoxInf || dx > 1024 || dilate_smem_bytes(r, dx, dilate_fused(r, dx)) > 200 * 1024;
}

inline void launch_dilate(const KParams& kp, int r, int streams, size_t /*smem*/, cudaStream_t st) {
  if (dilate_generic(r, kp.dx)) {
    for (int axis = 0; axis < 3; ++axis) {
      const long long len = axis == 0 ? kp.dx : (axis == 1 ? kp.dy : kp.dz);
      const long long lines = kp.n / len;
      const unsigned blocks = static_cast<unsigned>(std::min<long long>((lines + 255) / 256, 148LL * 8));
      launch_pdl(dilate_line_kernel, dim3(blocks, streams), dim3(256), 0, st, kp, r, axis);
    }
    return;
  }
  const int rows = kp.dy * kp.dz;
  const bool fused = dilate_fused(r, kp.dx);
  if (!fused) {
    // a single stream gets one row per warp-step of parallelism anyway; batches
    // amortise the per-warp setup over kDilRowsPerWarp rows
    const int G = dilate_rows_group(kp.dx);
    if (kp.n % 16 == 0 && G * kp.dx <= 512 && G * dilate_row_words(kp.dx) <= 32) {
      const int per_block = 8 * G;
      launch_pdl(dilate_rows_vec_kernel, dim3((rows + per_block - 1) / per_block, streams), dim3(256), 0, st, kp, r);
    } else {
      const int per_block = 8 * kDilRowsPerWarp;
      launch_pdl(dilate_rows_kernel, dim3((rows + per_block - 1) / per_block, streams), dim3(256), 0, st, kp, r);
    }
  }
  switch (r) {
    case 1: launch_dilate_tiles<1>(kp, r, fused, st, streams); break;
    case 2: launch_dilate_tiles<2>(kp, r, fused, st, streams); break;
    case 3: launch_dilate_tiles<3>(kp, r, fused, st, streams); break;
    case 4: launch_dilate_tiles<4>(kp, r, fused, st, streams); break;
    default: launch_dilate_tiles<0>(kp, r, fused, st, streams); break;
  }
}

// Opt-in to large dynamic shared memory for every K2b instance.
template <bool kFused, bool kClear>
inline cudaError_t dilate_set_smem_k(int bytes) {
  cudaError_t e = cudaSuccess;
  const void* fns[10] = {reinterpret_cast<const void*>(dilate_tiles_kernel<0, kFused, kClear>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<1, kFused, kClear>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<2, kFused, kClear>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<3, kFused, kClear>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<4, kFused, kClear>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<0, kFused, kClear, kDilTLone>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<1, kFused, kClear, kDilTLone>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<2, kFused, kClear, kDilTLone>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<3, kFused, kClear, kDilTLone>),
                         reinterpret_cast<const void*>(dilate_tiles_kernel<4, kFused, kClear, kDilTLone>)};
  for (const void* f : fns) {
    const cudaError_t x = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (x != cudaSuccess) e = x;
  }
  return e;
}
inline cudaError_t dilate_set_smem(int bytes) {
  cudaError_t e[4] = {dilate_set_smem_k<false, false>(bytes), dilate_set_smem_k<true, false>(bytes),
                      dilate_set_smem_k<false, true>(bytes), dilate_set_smem_k<true, true>(bytes)};
  for (cudaError_t x : e)
    if (x != cudaSuccess) return x;
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// K3: bundled frustum ray casting (paper Alg. 2): generate_rays
// (proj/src/raytracer.cpp:35-61) + walk_ray (proj/include/voxmap/raytracer.hpp:
// 76-118) + traverse_ray (raytracer.cpp:63-96). One thread per ray; a warp
// owns an 8x4 tile of end-plane targets so that its rays stay spatially
// coherent (lanes past the bundle's edge walk a clone of the edge ray).
//
// The walk runs in chunks of kChunk DDA steps: (A) the chunk's cell indices
// are computed (they do not depend on grid contents), (B) their occupancy
// bytes are loaded together through the read-only path, (C) the chunk is
// resolved in order with predicated PTX. Inside the grid each step only
// compares the chosen axis' tmax with a per-axis threshold min(stop, E_a),
// E_a the tmax at which the walk would leave the grid along a (decided by a
// value half a step below it), so there are no per-step bounds tests or step
// counters; chunks that provably cannot end any lane's walk skip even that
// (fast chunks), and chunks closer to the camera than any Occupied cell of
// the frame skip the occupancy loads (near field). ncu (profiles/) shows the
// kernel issue-bound, so the step and the resolve are written to minimise
// instructions per visit. The Sequential last-writer rule is a
// fire-and-forget RED.max on the cell key; before issuing it a lane drops its
// write when a higher lane (a higher ray index) writes the same cell in the
// same step, which removes most same-address traffic near the camera: over
// the whole warp with match.any, or against lane+1 and lane+8 with two
// shuffles (per step of a chunk, kMatchMask / kNearMask). Counters go to 32
// per-stream slots (one RED per warp each), summed by K4.
// ---------------------------------------------------------------------------

constexpr int kTraceSlots = 32;

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
// gvs is generate_rays' vox_size (direction and max_dist), vs the grid's
// (the walk): trace_bundle passes both (raytracer.cpp:100, 63-72).
__device__ __forceinline__ void ray_setup(const double* R, const FrameParams* fp, double vs,
                                          double gvs, int xi, int yi, int vd, RayState& st) {
  const double v0 = dmul(static_cast<double>(xi), gvs);
  const double v1 = dmul(static_cast<double>(yi), gvs);
  const double v2 = dmul(static_cast<double>(vd), gvs);
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#ifdef VXM_EIGEN34_MATVEC
    // Eigen 3.4's 3x3 * 3-vector: row 2 sums a0 + (a1 + a2) (see VoxmapEigenSubset.h)
    if (a == 2) {
      d[a] = dadd(dmul(R[3 * a], v0), dadd(dmul(R[3 * a + 1], v1), dmul(R[3 * a + 2], v2)));
      continue;
    }
#endif
    d[a] = dadd(dadd(dmul(R[3 * a], v0), dmul(R[3 * a + 1], v1)), dmul(R[3 * a + 2], v2));
  }
  const double xs = static_cast<double>(xi), ys = static_cast<double>(yi),
               ds = static_cast<double>(vd);
  const double max_dist = dmul(gvs, __dsqrt_rn(dadd(dadd(dmul(xs, xs), dmul(ys, ys)), dmul(ds, ds))));
  st.stop = dsub(max_dist, 1e-10);
  const double n2 = dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2]));
  const double nrm = __dsqrt_rn(n2);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double u = n2 > 0.0 ? ddiv(d[a], nrm) : d[a];
    // cur = floor(start / vs) and the numerators are per-frame constants
    // (set_ray_consts, the same IEEE operations on the host)
    st.cur[a] = fp->cam_cell[a];
    // u > 0: tmax = tnum_pos / u, tdelta = vs / u; u < 0: tnum_neg / u and
    // vs / -u; otherwise (0, NaN) both +inf. Written without branches (the
    // signs of u differ within a warp, the divisions run once): vs / |u| is
    // vs / u or vs / -u exactly, and the +inf select follows the divisions.
    const bool pos = u > 0.0, neg = u < 0.0;
    st.step[a] = pos ? 1 : (neg ? -1 : 0);
    const double tm = ddiv(pos ? fp->tnum_pos[a] : fp->tnum_neg[a], u);
    const double td = ddiv(vs, fabs(u));
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    st.tmax[a] = (pos || neg) ? tm : kInf;
    st.tdelta[a] = (pos || neg) ? td : kInf;
  }
}


// Two shapes (measured, tools/ab_time.sh): batches of frames run kChunk = 4
// steps per chunk in 2-warp blocks held to 48 registers (40 warps per SM;
// vxm_tuning.h), a lone frame (358 warps, GPU far from full) runs 8-step
// chunks in one-warp blocks at 64-80 registers, where per-warp latency
// decides, with each ray walked as two halves (kSplit) when it has few rays.
template <int kChunk, int kTraceWarps, int kMinBlocks, int kMatchMask, bool kFast, bool kSplit, int kNearMask = kMatchMask>
__global__ void __launch_bounds__(32 * kTraceWarps, kMinBlocks) trace_bundle_kernel(KParams p) {
  const int s = blockIdx.y;
  const FrameParams* fp = p.frames + s;
  const uint32_t epoch = fp->epoch;
  uint32_t* const key = fp->key_s;
  const uint8_t* const occ = fp->occ_s;
  double R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = fp->rot[i];

  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kTraceWarps + (threadIdx.x >> 5);
  const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
  // kSplit: a warp holds an 8x2 tile of rays twice, lanes 0-15 walking each
  // ray's near half (t < tau) and lanes 16-31 its far half
  const int rl = kSplit ? (lane & 15) : lane;
  const bool far_half = kSplit && lane >= 16;
  const int xi_idx = tx * 8 + (rl & 7);
  const int yi_idx = ty * (kSplit ? 2 : 4) + (rl >> 3);
  if (ty >= (kSplit ? (p.vh + 1) / 2 : p.tiles_y)) return;  // a whole warp past the bundle (block rounding)
  const bool active = xi_idx < p.vw && yi_idx < p.vh;
  // Lanes past the bundle's edge (partial edge tiles) walk a clone of the
  // edge ray, so that inside the grid every lane of a warp is live until its
  // ray ends: the clone makes the same cells, occupancy reads and keys as its
  // original (RED.max of equal keys, and the dedup keeps one of them), and
  // its counters are not added.
  const int xr = xi_idx < p.vw ? xi_idx : p.vw - 1, yr = yi_idx < p.vh ? yi_idx : p.vh - 1;
  const uint32_t ray = static_cast<uint32_t>(yr) * p.vw + xr;  // row-major, y outer
  const uint32_t ray_key = vxm::ray_key(p.key_fmt, epoch, ray);  // | 1: UnknownTraced

  RayState st;
  ray_setup(R, fp, p.vs, p.ray_vs, xr - (p.vw - 1) / 2, yr - (p.vh - 1) / 2, p.vd, st);
  // the ray setup above overlaps the tail of the populate/dilation kernels;
  // occupancy is read only from here on
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_trace = global_ns();
  // near field of the frame: every occupied cell lies at least near_dist from
  // the camera. A point P of the frame has |P| >= d (its depth; K1's bound),
  // its grid-frame image is within (1 +- 2e-6)|P| of the camera (R^T R is
  // within 1e-6 of I, pose_valid), and every cell of its dilated cube lies
  // within sqrt(3) (vox_inf + 1) vs of it; 1e-5 relative and 1e-6 m absolute
  // cover the rounding. 0 bits (not computed, e.g. a caller's grid with its
  // own Occupied cells) leave it negative.
  const double near_dist =
      dsub(dmul(static_cast<double>(__uint_as_float(__ldcg(&p.counters[s].min_dist_bits))), 1.0 - 1e-5),
           dadd(dmul(1.7320508075688774 * (p.vox_inf + 1) * (1.0 + 1e-9), p.vs), 1e-6));

  const unsigned dx = p.dx, dy = p.dy, dz = p.dz;
  const uint32_t dxy = dx * dy;
  // linear-index increment of one step along each axis; cell indices are
  // uint32 (grids of fewer than 2^32 cells) in modular arithmetic, exact for
  // every in-grid cell
  const uint32_t lin0 = static_cast<uint32_t>(st.step[0]), lin1 = static_cast<uint32_t>(st.step[1]) * dx,
                 lin2 = static_cast<uint32_t>(st.step[2]) * dxy;
  unsigned x = st.cur[0], y = st.cur[1], z = st.cur[2];
  uint32_t idx = static_cast<uint32_t>(st.cur[0]) + static_cast<uint32_t>(st.cur[1]) * dx +
                 static_cast<uint32_t>(st.cur[2]) * dxy;
  double t0 = st.tmax[0], t1 = st.tmax[1], t2 = st.tmax[2];
  const double stop = st.stop;

  bool walking = active && !far_half;  // (outside the grid a split warp walks whole rays on its near lanes)
  bool entered = false;
  unsigned freed = 0, traced = 0, skipped = 0;

  // Lean resolve (inline PTX, no branches but the RED's): per cell one
  // occupancy load, the write counter lw, the traced state carried in the
  // key itself (kv = ray_key | traced), snap = lw at the first occupied cell
  // (so traced writes = lw - snap at the end), the neighbour dedup through a
  // mask, and a predicated fire-and-forget RED.max on the key.
  uint32_t kv = ray_key;
  unsigned lw = 0, snap = 0xffffffffu;
  const unsigned long long key_base = reinterpret_cast<unsigned long long>(key);
#if VXM_TB_RED_HINT
  unsigned long long kpol;  // L2 evict-last on the keys K4 reads next
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(kpol));
#define VXM_RED_MAX(V, P) "@ok red.relaxed.gpu.global.max.L2::cache_hint.u32 [a], " V ", " P ";\n\t"
#define VXM_RED_POL , "l"(kpol)
#else
#define VXM_RED_MAX(V, P) "@ok red.relaxed.gpu.global.max.u32 [a], " V ";\n\t"
#define VXM_RED_POL
#endif
  // dedup bound: a cell is written when dup <= dup_max. With match.any, dup
  // is the mask of lanes on the same cell and no higher lane (higher ray
  // index) shares it exactly when dup <= lanemask_le (one compare instead of
  // an AND and a compare); the shuffle form gives dup in {0, 1}, bound 0.
  uint32_t dup_max = 0u;
  if constexpr ((kMatchMask | kNearMask) != 0) asm("mov.u32 %0, %%lanemask_le;" : "=r"(dup_max));

  // A write is dropped when a higher lane (higher ray index) makes the same
  // cell in the same step (measured: dropping the dedup after the first
  // chunks slows the kernel, the extra L2 atomics cost more than the check).
  // The lanes compare cells only: two lanes on the same cell read the same
  // occupancy byte, so either both write or neither does.
  // kTail: invalid cells only follow the end of the ray (the in-grid walk);
  // otherwise they can precede its entry into the grid (camera outside).
  // Two phases: prefetch issues the chunk's occupancy loads and dedup masks,
  // finish resolves the cells. (A software-pipelined walk that put the next
  // chunk's steps between them was measured slower: at 40 registers it
  // spills, at 64 the lower occupancy costs more than the latency it hides.)
  // the dedup of step j's cell c: the value the resolve compares with
  // dup_max (match mask, or 0/1 from the neighbour shuffles)
  auto dedup = [&](uint32_t c, int j, int mask = kMatchMask) -> uint32_t {
    uint32_t d;
    if ((mask >> j) & 1) {
      // the whole warp: only the highest lane of each distinct cell writes
      // (one match)
      asm("match.any.sync.b32 %0, %1, -1;" : "=r"(d) : "r"(c));
    } else {
      // lane+1 and lane+8 (two shuffles; the lone-frame kernel, whose serial
      // chain favours short latency)
      asm("{\n\t"
          ".reg .pred p1, p8, d1, d8;\n\t"
          ".reg .b32 r1, r8;\n\t"
          "shfl.sync.down.b32 r1|p1, %1, 1, %2, -1;\n\t"
          "shfl.sync.down.b32 r8|p8, %1, 8, %2, -1;\n\t"
          "setp.eq.and.u32 d1, r1, %1, p1;\n\t"
          "setp.eq.and.u32 d8, r8, %1, p8;\n\t"
          "or.pred d1, d1, d8;\n\t"
          "selp.u32 %0, 1, 0, d1;\n\t"
          "}"
          : "=r"(d)
          : "r"(c), "n"(kSplit ? 0x101f : 0x1f));  // kSplit: 16-lane segments (the halves)
    }
    return d;
  };
  // kLive: every cell of the chunk is valid (fast chunks: all lanes live).
  auto prefetch_t = [&](const uint32_t (&cell)[kChunk], uint32_t (&o)[kChunk], uint32_t (&dup)[kChunk],
                        auto tail_tag, auto live_tag) {
    constexpr bool kTail = decltype(tail_tag)::value;
    constexpr bool kLive = decltype(live_tag)::value;
#pragma unroll
    for (int j = 0; j < kChunk; ++j) {
      // a lane whose ray has ended reads as "occupied": no write, no count
      // (its traced state no longer matters; snap stays at or below its
      // final write count)
      if constexpr (kLive)
        o[j] = __ldg(occ + cell[j]);
      else
        o[j] = cell[j] != 0xffffffffu ? __ldg(occ + cell[j]) : (kTail ? epoch : 0u);
    }
    // the dedup first, for all cells of the chunk (it does not depend on the
    // loads, so its shuffle / match latency overlaps theirs): dup[j] >
    // dup_max when a higher lane makes the same cell in step j
#pragma unroll
    for (int j = 0; j < kChunk; ++j) dup[j] = dedup(cell[j], j);
  };
  auto finish_t = [&](const uint32_t (&cell)[kChunk], const uint32_t (&o)[kChunk], const uint32_t (&dup)[kChunk],
                      auto tail_tag) {
    constexpr bool kTail = decltype(tail_tag)::value;
#pragma unroll
    for (int j = 0; j < kChunk; ++j) {
// the per-cell resolve: predicates io (occupied) / w (write), the write
// count, snap, ok = w and no higher-lane duplicate, the RED.max of the key
// as it stands (a written cell is never occupied, so the traced bit, set
// after, cannot change at it), then the traced bit
#define VXM_RESOLVE_BODY                   \
  "@w add.u32 %1, %1, 1;\n\t"            \
  "@io min.u32 %2, %2, %1;\n\t"          \
  "setp.le.and.u32 ok, %7, %8, w;\n\t"   \
  "mul.wide.u32 a, %3, 4;\n\t"           \
  "add.u64 a, a, %6;\n\t"                \
  VXM_RED_MAX("%0", "%9") \
  "@io or.b32 %0, %0, 1;\n\t"
#define VXM_RESOLVE_DECL                   \
  ".reg .pred v, io, w, ok;\n\t"         \
  ".reg .b64 a;\n\t"
// kTail: the cell is valid or the ray has ended (o == epoch: no write)
#define VXM_RESOLVE_HEAD_TAIL "setp.eq.u32 io|w, %4, %5;\n\t"
// otherwise invalid cells (0xffffffff) may also precede the grid entry
#define VXM_RESOLVE_HEAD_ANY                \
  "setp.ne.u32 v, %3, -1;\n\t"            \
  "setp.eq.and.u32 io, %4, %5, v;\n\t"    \
  "setp.ne.and.u32 w, %4, %5, v;\n\t"
#define VXM_RESOLVE_ASM(HEAD)                                                    \
  asm volatile("{\n\t" VXM_RESOLVE_DECL HEAD VXM_RESOLVE_BODY "}"               \
               : "+r"(kv), "+r"(lw), "+r"(snap)                                  \
               : "r"(cell[j]), "r"(o[j]), "r"(epoch), "l"(key_base), "r"(dup[j]),                 \
                 "r"(((kMatchMask >> j) & 1) ? dup_max : 0u) VXM_RED_POL                           \
               : "memory")
      if constexpr (kTail)
        VXM_RESOLVE_ASM(VXM_RESOLVE_HEAD_TAIL);
      else
        VXM_RESOLVE_ASM(VXM_RESOLVE_HEAD_ANY);
#undef VXM_RESOLVE_ASM
#undef VXM_RESOLVE_HEAD_ANY
#undef VXM_RESOLVE_HEAD_TAIL
#undef VXM_RESOLVE_DECL
#undef VXM_RESOLVE_BODY
    }
  };
  auto resolve_t = [&](const uint32_t (&cell)[kChunk], auto tail_tag, auto live_tag) {
    uint32_t o[kChunk], dup[kChunk];
    prefetch_t(cell, o, dup, tail_tag, live_tag);
    finish_t(cell, o, dup, tail_tag);
  };
  auto resolve = [&](const uint32_t (&cell)[kChunk]) { resolve_t(cell, std::false_type{}, std::false_type{}); };
  // (kSplit: a near half's cells after its stop must not set its traced bit,
  // which the far half reads, so invalid cells take the general form)
  auto resolve_tail = [&](const uint32_t (&cell)[kChunk]) {
    if constexpr (kSplit)
      resolve_t(cell, std::false_type{}, std::false_type{});
    else
      resolve_t(cell, std::true_type{}, std::false_type{});
  };
  // every cell valid (a fast chunk): the tail form without the invalid-cell loads
  auto resolve_live = [&](const uint32_t (&cell)[kChunk]) { resolve_t(cell, std::true_type{}, std::true_type{}); };

  // The camera (every ray's start) is shared by the whole frame, so this
  // branch is uniform. Inside the grid the walk needs no per-cell bounds
  // test: it ends on the first step along an axis whose remaining in-grid
  // steps are used up.
  if (x < dx && y < dy && z < dz) {
    // The walk ends at the first step whose chosen axis a has tmax_a >= M_a,
    // M_a = min(stop, E_a), where E_a is the exact tmax_a value of the step
    // that would leave the grid along a (its rem_a-th step). So every step
    // checks one threshold and nothing else; no per-step bounds or counters.
    const int rem[3] = {st.step[0] > 0 ? static_cast<int>(dx - 1 - x) : static_cast<int>(x),
                        st.step[1] > 0 ? static_cast<int>(dy - 1 - y) : static_cast<int>(y),
                        st.step[2] > 0 ? static_cast<int>(dz - 1 - z) : static_cast<int>(z)};
    // E_a need not be summed: the walk's tmax values along a are strictly
    // increasing, T_a[k] ~ t_a + k tdelta_a, so "t_a >= E_a = T_a[rem_a]"
    // holds exactly when "t_a >= V" for any V in (T_a[rem_a - 1], T_a[rem_a]];
    // V = t_a + (rem_a - 1/2) tdelta_a is half a step away from both (the
    // rounding of k repeated adds is ~k 2^-53 of T, far below half a step),
    // and min(stop, V) decides every step exactly as min(stop, E_a) would.
    double M[3];
    const double tt[3] = {t0, t1, t2};
#pragma unroll
    for (int a = 0; a < 3; ++a)
      M[a] = st.step[a] != 0 ? fmin(stop, dadd(tt[a], dmul(static_cast<double>(rem[a]) - 0.5, st.tdelta[a]))) : stop;
    double M0 = M[0], M1 = M[1], M2 = M[2];
    // tdelta of an axis the ray never steps along is +inf; that axis is never
    // chosen, and the selected-addend form below needs a finite value for it
    // (and clamped to a finite value: the fast chunks add m * tdelta with
    // m in {0, 1}, which must leave t unchanged for m = 0; an axis whose
    // tdelta overflows is never chosen before the walk ends, and when it is
    // chosen at the walk's last step the sum no longer matters)
    constexpr double kMaxFinite = 0x1.fffffffffffffp+1023;
    const double e0 = st.step[0] ? fmin(st.tdelta[0], kMaxFinite) : 0.0,
                 e1 = st.step[1] ? fmin(st.tdelta[1], kMaxFinite) : 0.0,
                 e2 = st.step[2] ? fmin(st.tdelta[2], kMaxFinite) : 0.0;
    uint32_t al = 1u;  // every lane (clones included) walks a ray inside the grid
    // kSplit: the steps whose chosen tmax is below tau = min(M) / 2 (none of
    // which can end the walk) are the near half; its lane walks them with
    // every threshold at tau. The far lane starts where they end: along each
    // axis the tmax values below tau are taken with the walk's own repeated
    // additions, which gives that axis' step count and the exact tmax.
    double fs0 = 0.0, fs1 = 0.0, fs2 = 0.0;  // the far half's start, for its re-walk
    uint32_t fidx = 0;
    if constexpr (kSplit) {
      const double tau = dmul(0.5, fmin(fmin(M0, M1), M2));
      if (!far_half) {
        M0 = M1 = M2 = tau;
      } else {
        while (t0 < tau) { t0 = dadd(t0, e0); idx += lin0; }
        while (t1 < tau) { t1 = dadd(t1, e1); idx += lin1; }
        while (t2 < tau) { t2 = dadd(t2, e2); idx += lin2; }
        fs0 = t0; fs1 = t1; fs2 = t2;
        fidx = static_cast<uint32_t>(idx);
      }
    }
    uint32_t uidx = static_cast<uint32_t>(idx);
    // Fast chunks (kFast): the walk ends at a step whose chosen tmax reaches
    // its axis' threshold M_a >= min(M). Within the next kChunk steps every
    // chosen tmax is at most min_a(t_a + (kChunk-1) tdelta_a): were axis b
    // that minimum, each step takes the current minimum, which is at most
    // b's current value, and b advances at most kChunk-1 times before the
    // last step. So while that bound (an fma, one rounding; the walk's
    // repeated adds stay within (kChunk+1) 2^-53 of it) is below lim =
    // min(M)(1 - 2^-40), no step of the chunk can end the walk: the chunk
    // runs without threshold tests, and with every lane live its cells are
    // all valid (no invalid-cell handling in the resolve). The warp takes
    // it when all lanes qualify (~80% of a cfg2 bundle's chunks).
    const double Mmin = fmin(fmin(M0, M1), M2);
    constexpr double kAhead = static_cast<double>(kChunk - 1);
    // kChunk exact steps (threshold tests included), their cells into cell[]
    auto step_chunk = [&](uint32_t (&cell)[kChunk]) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        cell[j] = al ? uidx : 0xffffffffu;
        // walk_ray's step (raytracer.hpp:103-116): the axis with the smallest
        // tmax, ties x then y then z; the walk goes on while that tmax is
        // below its threshold. t + 0 == t for the axes not taken (t >= 0).
        asm("{\n\t"
            ".reg .pred q, px, py, pz, npx, s0, s1, s2, ok;\n\t"
            ".reg .f64 a0, a1, a2;\n\t"
            ".reg .b32 l;\n\t"
            "setp.le.f64 q, %0, %1;\n\t"
            "setp.le.and.f64 px, %0, %2, q;\n\t"
            "setp.le.f64 q, %1, %2;\n\t"
            "not.pred npx, px;\n\t"
            "and.pred py, q, npx;\n\t"
            "or.pred pz, px, py;\n\t"
            "not.pred pz, pz;\n\t"
            "setp.lt.and.f64 s0, %0, %8, px;\n\t"
            "setp.lt.and.f64 s1, %1, %9, py;\n\t"
            "setp.lt.and.f64 s2, %2, %10, pz;\n\t"
            "or.pred ok, s0, s1;\n\t"
            "or.pred ok, ok, s2;\n\t"
            "selp.u32 %4, %4, 0, ok;\n\t"
            // t_a = fma(m_a, e_a, t_a), m_a in {0, 1} (as in the fast chunks)
            "selp.f64 a0, 0d3FF0000000000000, 0d0000000000000000, px;\n\t"
            "selp.f64 a1, 0d3FF0000000000000, 0d0000000000000000, py;\n\t"
            "selp.f64 a2, 0d3FF0000000000000, 0d0000000000000000, pz;\n\t"
            "fma.rn.f64 %0, a0, %5, %0;\n\t"
            "fma.rn.f64 %1, a1, %6, %1;\n\t"
            "fma.rn.f64 %2, a2, %7, %2;\n\t"
            "selp.b32 l, %12, %13, py;\n\t"
            "selp.b32 l, %11, l, px;\n\t"
            "add.s32 %3, %3, l;\n\t"
            "}"
            : "+d"(t0), "+d"(t1), "+d"(t2), "+r"(uidx), "+r"(al)
            : "d"(e0), "d"(e1), "d"(e2), "d"(M0), "d"(M1), "d"(M2), "r"(lin0), "r"(lin1), "r"(lin2));
        // the near half stops at tau without recording that cell: it is the
        // far half's first
        if (kSplit && !far_half && !al) cell[j] = 0xffffffffu;
      }
    };
    // lim = -inf once the lane's walk has ended (set after the exact chunk
    // it ends in), so the fast test needs no liveness term
    double lim = dsub(Mmin, dmul(0x1p-40, fabs(Mmin)));
    // the fast-chunk test against a limit: some axis of every lane has
    // fma(kChunk-1, tdelta_a, t_a) below it (PTX compares chained with or:
    // left to ptxas, the three compares become an fmin with NaN handling)
    auto fast_test = [&](double lm, double ahead = static_cast<double>(kChunk - 1)) -> uint32_t {
      uint32_t ok = 0;
      asm("{\n\t"
          ".reg .pred p;\n\t"
          ".reg .f64 b;\n\t"
          "fma.rn.f64 b, %1, %2, %3;\n\t"
          "setp.lt.f64 p, b, %8;\n\t"
          "fma.rn.f64 b, %1, %4, %5;\n\t"
          "setp.lt.or.f64 p, b, %8, p;\n\t"
          "fma.rn.f64 b, %1, %6, %7;\n\t"
          "setp.lt.or.f64 p, b, %8, p;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t"
          "}"
          : "=r"(ok)
          : "d"(ahead), "d"(e0), "d"(t0), "d"(e1), "d"(t1), "d"(e2), "d"(t2), "d"(lm));
      return ok;
    };
    // two chunks under one test (the same bound with 2 kChunk - 1 steps ahead)
    constexpr bool kFast2 = VXM_TB_FAST2 && kTraceWarps > 1;
    constexpr double kAhead2 = static_cast<double>(2 * kChunk - 1);
    // kChunk steps without threshold tests: t_a = fma(m_a, e_a, t_a) with
    // m_a = 1 on the chosen axis, 0 elsewhere (fma(1, e, t) = RN(t + e),
    // fma(0, e, t) = t), one select of a high word per axis
    auto fast_steps = [&](uint32_t (&cell)[kChunk]) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        cell[j] = uidx;
        asm("{\n\t"
            ".reg .pred q, px, py, pxy;\n\t"
            ".reg .f64 m0, m1, m2;\n\t"
            ".reg .b32 l;\n\t"
            "setp.le.f64 q, %0, %1;\n\t"
            "setp.le.and.f64 px, %0, %2, q;\n\t"
            "setp.le.f64 q, %1, %2;\n\t"
            "and.pred py, q, !px;\n\t"
            "or.pred pxy, px, py;\n\t"
            "selp.f64 m0, 0d3FF0000000000000, 0d0000000000000000, px;\n\t"
            "selp.f64 m1, 0d3FF0000000000000, 0d0000000000000000, py;\n\t"
            "selp.f64 m2, 0d0000000000000000, 0d3FF0000000000000, pxy;\n\t"
            "fma.rn.f64 %0, m0, %4, %0;\n\t"
            "fma.rn.f64 %1, m1, %5, %1;\n\t"
            "fma.rn.f64 %2, m2, %6, %2;\n\t"
            "selp.b32 l, %8, %9, py;\n\t"
            "selp.b32 l, %7, l, px;\n\t"
            "add.s32 %3, %3, l;\n\t"
            "}"
            : "+d"(t0), "+d"(t1), "+d"(t2), "+r"(uidx)
            : "d"(e0), "d"(e1), "d"(e2), "r"(lin0), "r"(lin1), "r"(lin2));
      }
    };
    if constexpr (kFast) {
      // Near field: a step whose chosen tmax (the cell's exit) is below
      // near_dist leaves a cell no occupied cell can be, so while the chunk
      // bound is below min(lim, near_dist) for every lane the chunk needs no
      // occupancy loads: every cell is written (untraced state unchanged),
      // only the dedup and the RED remain.
      const double lim_near = fmin(lim, near_dist);
      int near_reps = 1;  // chunks per test: 2 while the two-chunk bound holds
      if constexpr (kFast2) near_reps = __all_sync(0xffffffffu, fast_test(lim_near, kAhead2)) ? 2 : 1;
      while (near_reps == 2 || __all_sync(0xffffffffu, fast_test(lim_near))) {
        for (int rep = 0; rep < near_reps; ++rep) {
        uint32_t cell[kChunk];
        fast_steps(cell);
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
          const uint32_t dup = dedup(cell[j], j, kNearMask);
          asm volatile("{\n\t.reg .pred ok;\n\t.reg .b64 a;\n\t"
                       "setp.le.u32 ok, %1, %2;\n\t"
                       "mul.wide.u32 a, %0, 4;\n\t"
                       "add.u64 a, a, %3;\n\t"
                       VXM_RED_MAX("%4", "%5") "}"
                       :: "r"(cell[j]), "r"(dup), "r"(((kNearMask >> j) & 1) ? dup_max : 0u), "l"(key_base), "r"(kv)
                          VXM_RED_POL
                       : "memory");
        }
        lw += kChunk;
        }
        if constexpr (kFast2) near_reps = __all_sync(0xffffffffu, fast_test(lim_near, kAhead2)) ? 2 : 1;
      }
    }
    // (the one-warp kernel only: in the 48-register batch kernel the extra
    // code lengthened the all-live fast chunk, r02ch)
    constexpr bool kTailFast = VXM_TB_TAIL_FAST && kTraceWarps == 1;
    if constexpr (kTailFast) {
    // Once some lanes' walks have ended (only an exact chunk ends one), their
    // lim is +inf, so they never block a fast chunk: the warp's tail takes
    // fast chunks whenever its live lanes qualify, with the ended lanes' cells
    // masked (they keep stepping; an invalid cell reads as occupied: no write,
    // no count) instead of exact chunks to the end of its longest ray.
    bool all_live = true;  // (warp-uniform)
    for (;;) {
      if (kFast && __all_sync(0xffffffffu, fast_test(lim))) {
        uint32_t cell[kChunk];
        fast_steps(cell);
        if (all_live) {
          resolve_live(cell);
        } else {
#pragma unroll
          for (int j = 0; j < kChunk; ++j) cell[j] = al ? cell[j] : 0xffffffffu;
          resolve_tail(cell);
        }
        continue;
      }
      uint32_t cell[kChunk];
      step_chunk(cell);
      resolve_tail(cell);
      if (!al) lim = __longlong_as_double(0x7ff0000000000000ll);
      const unsigned live = __ballot_sync(0xffffffffu, al != 0u);
      if (!live) break;
      all_live = live == 0xffffffffu;
    }
    } else {
#if VXM_TB_TAIL_FAST_BATCH
    // the batch kernel: the all-live fast loop as below, and the masked fast
    // chunk tried only where the tail would take an exact chunk (lim2 = lim of
    // the live lanes, +inf for the ended ones)
    double lim2 = lim;
    for (;;) {
      if (kFast && __all_sync(0xffffffffu, fast_test(lim))) {
        uint32_t cell[kChunk];
        fast_steps(cell);
        resolve_live(cell);
        continue;
      }
      if (!__any_sync(0xffffffffu, al != 0u)) break;
      if (kFast && __all_sync(0xffffffffu, fast_test(lim2))) {
        uint32_t cell[kChunk];
        fast_steps(cell);
#pragma unroll
        for (int j = 0; j < kChunk; ++j) cell[j] = al ? cell[j] : 0xffffffffu;
        resolve_tail(cell);
        continue;
      }
      uint32_t cell[kChunk];
      step_chunk(cell);
      resolve_tail(cell);
      if (!al) {
        lim = -__longlong_as_double(0x7ff0000000000000ll);
        lim2 = __longlong_as_double(0x7ff0000000000000ll);
      }
    }
#else
    for (;;) {
      if (kFast2 && __all_sync(0xffffffffu, fast_test(lim, kAhead2))) {
#pragma unroll 1
        for (int rep = 0; rep < 2; ++rep) {
          uint32_t cell[kChunk];
          fast_steps(cell);
          resolve_live(cell);
        }
        continue;
      }
      if (kFast && __all_sync(0xffffffffu, fast_test(lim))) {
        uint32_t cell[kChunk];
        fast_steps(cell);
        resolve_live(cell);
        continue;
      }
      if (!__any_sync(0xffffffffu, al != 0u)) break;
      uint32_t cell[kChunk];
      step_chunk(cell);
      resolve_tail(cell);
      if (!al) lim = -__longlong_as_double(0x7ff0000000000000ll);
    }
#endif
    }
    if constexpr (kSplit) {
      // The far half resolved its cells as if nothing before it were
      // occupied. If the near half met an occupied cell, the far half's writes
      // before its own first occupied cell (min(snap, lw) of them, all
      // unoccupied) carry the traced bit: count them so and write their keys
      // again with it (RED.max: the higher key wins), walking that prefix once
      // more. (A clone's original does this for it.)
      const uint32_t near_traced = __shfl_sync(0xffffffffu, kv & 1u, lane & 15);
      if (far_half && active && near_traced) {
        unsigned n = min(snap, lw);
        snap = 0;
        double a0 = fs0, a1 = fs1, a2 = fs2;
        uint32_t u = fidx;
        const uint32_t kt = ray_key | 1u;
        for (; n > 0; --n) {
          atomicMax(key + u, kt);
          const bool bx = a0 <= a1 && a0 <= a2;
          const bool by = !bx && a1 <= a2;
          if (bx) { a0 = dadd(a0, e0); u += lin0; }
          else if (by) { a1 = dadd(a1, e1); u += lin1; }
          else { a2 = dadd(a2, e2); u += lin2; }
        }
      }
    }
  } else {
  while (__any_sync(0xffffffffu, walking)) {
    uint32_t cell[kChunk];
#pragma unroll
    for (int j = 0; j < kChunk; ++j) {
      const bool inb = x < dx && y < dy && z < dz;
      const bool visit = walking && inb;
      skipped += (walking && !inb && !entered) ? 1u : 0u;
      walking = walking && (inb || !entered);  // a line leaves a convex grid exactly once
      entered = entered || visit;
      cell[j] = visit ? static_cast<uint32_t>(idx) : 0xffffffffu;
      // walk_ray's step (raytracer.hpp:103-116): ties step x, then y, then z
      const bool bx = t0 <= t1 && t0 <= t2;
      const bool by = !bx && t1 <= t2;
      const double tm = bx ? t0 : (by ? t1 : t2);
      walking = walking && !(tm >= stop);
      if (walking) {
        if (bx) {
          t0 = dadd(t0, st.tdelta[0]);
          x += st.step[0];
          idx += lin0;
        } else if (by) {
          t1 = dadd(t1, st.tdelta[1]);
          y += st.step[1];
          idx += lin1;
        } else {
          t2 = dadd(t2, st.tdelta[2]);
          z += st.step[2];
          idx += lin2;
        }
      }
    }
    resolve(cell);
  }
  }
  // writes before the first occupied cell free, the rest are traced; a
  // clone's counts belong to its original
  if (active) {
    freed = min(snap, lw);
    traced = lw - freed;
  }
  unsigned long long* slot = &p.counters[s].trace_slots[tile % kTraceSlots][0];
  const unsigned r_n = __reduce_add_sync(0xffffffffu, active && !far_half ? 1u : 0u);
  const unsigned f_n = __reduce_add_sync(0xffffffffu, freed);
  const unsigned t_n = __reduce_add_sync(0xffffffffu, traced);
  const unsigned k_n = __reduce_add_sync(0xffffffffu, skipped);
  if (lane == 0) {
    if (r_n) atomicAdd(slot + 0, r_n);
    if (f_n) atomicAdd(slot + 1, f_n);
    if (t_n) atomicAdd(slot + 2, t_n);
    if (k_n) atomicAdd(slot + 3, k_n);
  }
}

// Launches K3 over `slots` frame slots in the shape that suits the batch.
constexpr long long kSplitMaxRays = VXM_TB_SPLIT_MAX_RAYS;
// batch K3 shape: VXM_TB_* (vxm_tuning.h)

// `batch` is the number of slots of the whole call (graph branches launch
// shares of it concurrently, so the GPU is as full as the total says).
inline void launch_trace(const KParams& kp, int slots, int batch, cudaStream_t st) {
  const int tiles = kp.tiles_x * kp.tiles_y;
  if (batch >= VXM_TB_BATCH_MIN) {
    // dedup by match.any on every step for large bundles, on every other step
    // (shuffles between) for small ones (VXM_TB_MATCH_* in vxm_tuning.h)
    const dim3 grid((tiles + VXM_TB_WARPS - 1) / VXM_TB_WARPS, slots), block(32 * VXM_TB_WARPS);
    if (static_cast<long long>(kp.vw) * kp.vh >= VXM_TB_MATCH_RAYS)
      launch_pdl(trace_bundle_kernel<VXM_TB_CHUNK, VXM_TB_WARPS, VXM_TB_MINB, VXM_TB_MATCH_LARGE, VXM_TB_FAST, false, VXM_TB_NEAR_MATCH_LARGE>,
                 grid, block, 0, st, kp);
    else
      launch_pdl(trace_bundle_kernel<VXM_TB_CHUNK, VXM_TB_WARPS, VXM_TB_MINB, VXM_TB_MATCH_SMALL, VXM_TB_FAST, false, VXM_TB_NEAR_MATCH_SMALL>,
                 grid, block, 0, st, kp);
  } else {
    if (static_cast<long long>(kp.vw) * kp.vh * batch <= kSplitMaxRays) {
      // few rays (the GPU far from full): 8x2 tiles, each ray walked as two
      // halves by two lanes; measured -12% / -7% K3 time for a lone cfg2 /
      // cfg1 frame, +11% for a lone cfg3 frame (76k rays)
      const int tiles2 = kp.tiles_x * ((kp.vh + 1) / 2);
      launch_pdl(trace_bundle_kernel<8, 1, 1, 0, true, true>, dim3(tiles2, slots), dim3(32), 0, st, kp);
    } else {
      launch_pdl(trace_bundle_kernel<8, 1, 1, 0, true, false>, dim3(tiles, slots), dim3(32), 0, st, kp);
    }
  }
}

// Sums K3's per-slot counters into the stream's totals (one warp).
__device__ __forceinline__ void fold_trace_slots(Counters& c) {
  const int lane = threadIdx.x & 31;
  unsigned long long v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = c.trace_slots[lane][i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], o);
  }
  if (lane == 0) {
    c.rays_traced = v[0];
    c.voxels_freed = v[1];
    c.voxels_traced = v[2];
    c.voxels_skipped = v[3];
  }
}

// ---------------------------------------------------------------------------
// K3b: the per-pixel comparison tracer (TracerMode::PerPixelBaseline, paper
// §V-D): bresenham_trace_image (proj/src/raytracer.cpp:120-161) with
// bresenham_line (proj/include/voxmap/raytracer.hpp:136-194). One thread per
// cloud point (or per depth pixel, back-projected again exactly as K1 does).
// Every write stores Free and occupancy is frozen during the trace, so the
// Sequential result is order independent: plain stores, no atomics. Free is
// written as a key with ray index 0 (decodes to Free).
// ---------------------------------------------------------------------------
struct PerPixelAcc {
  unsigned rays, freed, skipped;
};

__device__ __forceinline__ void pp_visit(const KParams& p, const int* c, const int* end,
                                         const uint8_t* occ, uint32_t* key, uint32_t epoch,
                                         PerPixelAcc& acc) {
  if (c[0] == end[0] && c[1] == end[1] && c[2] == end[2]) return;  // the endpoint holds the obstacle
  if (static_cast<unsigned>(c[0]) >= static_cast<unsigned>(p.dx) ||
      static_cast<unsigned>(c[1]) >= static_cast<unsigned>(p.dy) ||
      static_cast<unsigned>(c[2]) >= static_cast<unsigned>(p.dz)) {
    ++acc.skipped;
    return;
  }
  const uint32_t idx = static_cast<uint32_t>(c[0]) + static_cast<uint32_t>(c[1]) * p.dx +
                       static_cast<uint32_t>(c[2]) * (static_cast<uint32_t>(p.dx) * static_cast<uint32_t>(p.dy));
  if (occ[idx] != epoch) {
    // Free (every per-pixel write stores the same lowest-priority Free key)
    key[idx] = ray_key(p.key_fmt, epoch, -1);
    ++acc.freed;
  }
}

__device__ __forceinline__ void pp_trace_point(const KParams& p, const double* R, const double* t,
                                               const int* cam, double x, double y, double z,
                                               const uint8_t* occ, uint32_t* key, uint32_t epoch,
                                               PerPixelAcc& acc) {
  // world_to_voxel(t_vc.apply(point)) (grid.cpp:54-62, geometry.cpp:10-15):
  // ((R p) + t) / vs, rows left to right, floor, int
  int end[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double w = dadd(dadd(dadd(dmul(R[3 * a], x), dmul(R[3 * a + 1], y)), dmul(R[3 * a + 2], z)), t[a]);
    end[a] = static_cast<int>(floor(ddiv(w, p.vs)));
  }
  ++acc.rays;
  int q[3] = {cam[0], cam[1], cam[2]};
  int d[3], sg[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    d[a] = abs(end[a] - q[a]);
    sg[a] = end[a] > q[a] ? 1 : -1;
  }
  int drive, o1, o2;
  if (d[0] >= d[1] && d[0] >= d[2]) {
    drive = 0; o1 = 1; o2 = 2;
  } else if (d[1] >= d[0] && d[1] >= d[2]) {
    drive = 1; o1 = 0; o2 = 2;
  } else {
    drive = 2; o1 = 1; o2 = 0;
  }
  int p1 = 2 * d[o1] - d[drive], p2 = 2 * d[o2] - d[drive];
  while (q[drive] != end[drive]) {
    pp_visit(p, q, end, occ, key, epoch, acc);
    if (p1 >= 0) { q[o1] += sg[o1]; p1 -= 2 * d[drive]; }
    if (p2 >= 0) { q[o2] += sg[o2]; p2 -= 2 * d[drive]; }
    p1 += 2 * d[o1];
    p2 += 2 * d[o2];
    q[drive] += sg[drive];
  }
  // the final visit(to) of bresenham_line is the endpoint: skipped by pp_visit
}

// from_depth: pixels of fp->depth (back-projected as K1), else fp->xs/ys/zs.
__global__ void __launch_bounds__(256) trace_per_pixel_kernel(KParams p, int from_depth) {
  pdl_wait();
  const int s = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_trace = global_ns();
  const FrameParams* fp = p.frames + s;
  const uint32_t epoch = fp->epoch;
  uint32_t* const key = p.key + static_cast<long long>(s) * p.n;
  const uint8_t* occ = p.occ + static_cast<long long>(s) * p.n;
  double R[9], t[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = fp->rot[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = fp->trans[i];
  int cam[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) cam[a] = static_cast<int>(floor(ddiv(t[a], p.vs)));
  PerPixelAcc acc{0, 0, 0};
  const long long n = from_depth ? static_cast<long long>(p.W) * p.H : fp->n_points;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double x, y, z;
    if (from_depth) {
      const float d = fp->depth[i];
      if (!(isfinite(d) && d > 0.0f)) continue;
      z = static_cast<double>(d);
      if (z > p.max_depth) continue;
      const int v = static_cast<int>(i / p.W), u = static_cast<int>(i - static_cast<long long>(v) * p.W);
      x = dmul(__ldg(p.qx + u), z);
      y = dmul(__ldg(p.qy + v), z);
    } else {
      x = fp->xs[i];
      y = fp->ys[i];
      z = fp->zs[i];
      if (!(isfinite(x) && isfinite(y) && isfinite(z))) continue;
    }
    pp_trace_point(p, R, t, cam, x, y, z, occ, key, epoch, acc);
  }
  unsigned vals[3] = {acc.rays, acc.freed, acc.skipped};
  unsigned long long* dst[3] = {&p.counters[s].trace_slots[blockIdx.x % 32][0],
                                &p.counters[s].trace_slots[blockIdx.x % 32][1],
                                &p.counters[s].trace_slots[blockIdx.x % 32][3]};
  block_accumulate<3>(vals, dst);
}

// ---------------------------------------------------------------------------
// K4: merge_grids (proj/src/pipeline.cpp:44-61) + shift_grid_by
// (proj/src/grid.cpp:81-108) + the two VoxelGrid::count passes
// (pipeline.cpp:114-115) in one gather: destination cell c takes
// merge(loc[c+off], ms[c+off]) when c+off is inside the grid, else Unknown.
// Reads the current local buffer, writes the other (ping-pong). One warp per
// x-row (rows_per_warp rows per warp: 1 for a single stream, up to
// kRowsPerWarp when a batch fills the GPU); each lane produces 4 cells.
// When dx and the x-shift are multiples of 4 (all benchmark grids), the 4
// cells move as one 32-bit word and are decoded / merged with byte-SIMD
// intrinsics; otherwise a per-cell path runs.
// ---------------------------------------------------------------------------
constexpr int kRowsPerWarp = 4;

// K5: after K4, one block per slot copies the slot's counters to the
// host-mapped read-back buffer and zeroes them, K3's per-warp partials
// included, for the next frame (so the frame graph has neither a memset nor
// a D2H copy node; a last-block check-in inside K4 cost its ~10k blocks more
// than this launch).
// K5's work for slot s: the counters into host-mapped memory, then cleared
// (K3's partials included) for the next frame. Device function: K5 runs it in
// one block per slot, or the last K4 block of a slot runs it (publish_when_last).
// (threads t0 .. t0 + nt - 1 of the block take part)
// clears slot s's counters for the next frame (threads t of nt)
__device__ __forceinline__ void publish_slot_clear(const KParams& p, int s, int t, int nt) {
  constexpr int kHead = sizeof(CountersHead) / sizeof(unsigned long long);
  constexpr int kParts = sizeof(Counters::trace_slots) / sizeof(unsigned long long);
  unsigned long long* c = reinterpret_cast<unsigned long long*>(p.counters + s);
  if (t < kHead) c[t] = 0ull;
  for (int i = t; i < kParts; i += nt) (&p.counters[s].trace_slots[0][0])[i] = 0ull;
  if (t == 0) {
    p.counters[s].merge_done = 0ull;
    p.counters[s].min_dist_bits = 0x7F800000u;
    p.counters[s].pop_faces = (p.counters[s].pop_faces & 0xFFFFu) << 16;
  }
}
__device__ __forceinline__ void publish_slot(const KParams& p, int s, int t = threadIdx.x, int nt = blockDim.x) {
  constexpr int kHead = sizeof(CountersHead) / sizeof(unsigned long long);
  unsigned long long* c = reinterpret_cast<unsigned long long*>(p.counters + s);
  if (t < kHead) reinterpret_cast<unsigned long long*>(p.counters_out + s)[t] = __ldcg(c + t);
  __syncwarp();  // (t < 32 here: the copies precede the clearing)
  publish_slot_clear(p, s, t, nt);
}

// End of a K4 block: the slot's last block to finish publishes its counters
// (threadfence reduction: every block's counter atomics are ordered before its
// increment of merge_done), so no K5 launch follows K4.
// Only warp 0 takes part (it made the block's counter atomics); the other
// warps leave without waiting for the fence.
__device__ __forceinline__ void publish_when_last(const KParams& p, int s) {
  if (threadIdx.x >= 32) return;
  unsigned last = 0;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&p.counters[s].merge_done, 1ull) == gridDim.x - 1 ? 1u : 0u;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  publish_slot(p, s, threadIdx.x, 32);
}

// The packed publish of K4 (grids below 2^24 cells, fewer than 2^16 blocks per
// slot): each block adds (1 << 48 | freed << 24 | occupied) to merge_done; the
// block that brings the count to gridDim.x holds the totals in the returned
// value, folds K3's partials (written by the previous kernel, so visible) and
// publishes. Only block 0 fences (so that its t_merge stamp is visible first).
__device__ __forceinline__ void publish_packed(const KParams& p, int s, unsigned occ_n, unsigned free_n) {
  __shared__ unsigned long long part[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const unsigned o = __reduce_add_sync(0xffffffffu, occ_n), f = __reduce_add_sync(0xffffffffu, free_n);
  if (lane == 0) {
    part[0][warp] = o;
    part[1][warp] = f;
  }
  __syncthreads();
  if (warp != 0) return;
  unsigned long long bo = lane < nw ? part[0][lane] : 0ull, bf = lane < nw ? part[1][lane] : 0ull;
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) {
    bo += __shfl_down_sync(0xffffffffu, bo, k);
    bf += __shfl_down_sync(0xffffffffu, bf, k);
  }
  unsigned long long tot = 0;
  unsigned last = 0;
  if (lane == 0) {
    if (blockIdx.x == 0) __threadfence();
    const unsigned long long add = (1ull << 48) | (bf << 24) | bo;
    tot = atomicAdd(&p.counters[s].merge_done, add) + add;
    last = (tot >> 48) == gridDim.x ? 1u : 0u;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  tot = __shfl_sync(0xffffffffu, tot, 0);
  __threadfence();  // (acquire side: block 0's t_merge)
  Counters& c = p.counters[s];
  unsigned long long v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = __ldcg(&c.trace_slots[lane][i]);
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], k);
  }
  if (lane == 0) {
    CountersHead h;
    h.points_total = __ldcg(&c.points_total);
    h.points_outside = __ldcg(&c.points_outside);
    h.rays_traced = v[0];
    h.voxels_freed = v[1];
    h.voxels_traced = v[2];
    h.voxels_skipped = v[3];
    h.occupied = tot & 0xFFFFFFull;
    h.freed = (tot >> 24) & 0xFFFFFFull;
    h.t_pop = __ldcg(&c.t_pop);
    h.t_trace = __ldcg(&c.t_trace);
    h.t_merge = __ldcg(&c.t_merge);
    h.t_end = global_ns();
    p.counters_out[s] = h;
  }
  __syncwarp();
  publish_slot_clear(p, s, lane, 32);
}

__global__ void __launch_bounds__(128) publish_counters_kernel(KParams p) {
  pdl_wait();  // K4 complete
  publish_slot(p, blockIdx.x);
}

// number of bytes of x (states 0..3) equal to 2 / to 1
__device__ __forceinline__ unsigned count_occupied4(uint32_t x) { return __popc((x >> 1) & ~x & 0x01010101u); }
__device__ __forceinline__ unsigned count_free4(uint32_t x) { return __popc(x & ~(x >> 1) & 0x01010101u); }

// floor(a / d) for a < 2^24 with a fp32 reciprocal and one correction (the
// estimate is off by at most one there)
__device__ __forceinline__ uint32_t div_small(uint32_t a, uint32_t d, float inv_d) {
  uint32_t q = __float2uint_rz(__uint2float_rn(a) * inv_d);
  const int r = static_cast<int>(a) - static_cast<int>(q * d);
  q = r < 0 ? q - 1 : q;
  return r >= static_cast<int>(d) ? q + 1 : q;
}

// number of bytes equal to 2 / to 1 over four words of states (byte sums of
// the per-byte flags, each at most 4, gathered by one multiply)
__device__ __forceinline__ unsigned count_occupied16(const uint32_t (&x)[4]) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) m += (x[i] >> 1) & ~x[i] & 0x01010101u;
  return (m * 0x01010101u) >> 24;
}
__device__ __forceinline__ unsigned count_free16(const uint32_t (&x)[4]) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) m += x[i] & ~(x[i] >> 1) & 0x01010101u;
  return (m * 0x01010101u) >> 24;
}

// merge of 4 packed cells: local l4, occupancy o4 (epoch bytes), 4 epoch keys.
// States are 0..3 per byte, so "== 0" and "== 3" are two-bit tests.
__device__ __forceinline__ uint32_t merge4(uint32_t l4, uint32_t o4, uint4 k4, uint32_t epoch) {
#if VXM_MERGE4_PRMT
  // the four keys' bytes 3, 2 and 0 gathered into one word each (byte i =
  // key i's byte): a key is this frame's iff byte 3 == epoch >> 6 and the top
  // six bits of byte 2 == epoch & 63 (epoch << 18, 14 bits); bit 0 of byte 0
  // is its traced bit
  static_assert(kKeyShift == 18, "byte layout of the epoch keys");
  const uint32_t b3 = __byte_perm(__byte_perm(k4.x, k4.y, 0x0073), __byte_perm(k4.z, k4.w, 0x0073), 0x5410);
  const uint32_t b2 = __byte_perm(__byte_perm(k4.x, k4.y, 0x0062), __byte_perm(k4.z, k4.w, 0x0062), 0x5410);
  const uint32_t b0 = __byte_perm(__byte_perm(k4.x, k4.y, 0x0040), __byte_perm(k4.z, k4.w, 0x0040), 0x5410);
  const uint32_t e3 = ((epoch >> 6) & 0xffu) * 0x01010101u, e2 = ((epoch & 63u) << 2) * 0x01010101u;
  const uint32_t valid = zero_bytes((b3 ^ e3) | ((b2 & 0xfcfcfcfcu) ^ e2));  // 0xff per key of this frame
  uint32_t m4 = valid & (0x01010101u | ((b0 << 1) & 0x02020202u));            // 1 or 3
#else
  const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
  uint32_t m4 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t v = (kk[i] >> kKeyShift) == epoch ? (1u | ((kk[i] & 1u) << 1)) : 0u;  // 1 or 3
    m4 |= v << (8 * i);
  }
#endif
  const uint32_t occm = zero_bytes(o4 ^ (epoch * 0x01010101u));  // 0xff where Occupied
  m4 = (m4 & ~occm) | (0x02020202u & occm);
  const uint32_t keep = (((m4 | (m4 >> 1)) & 0x01010101u) ^ 0x01010101u) * 0xffu;  // m == 0
  const uint32_t clear = (m4 & (m4 >> 1) & 0x01010101u) * 0xffu;                   // m == 3
  return (l4 & keep) | (m4 & ~(keep | clear));
}

// K4, epoch-format keys (every bundle of up to 131,070 rays): merge4 decodes
// occupancy bytes and keys; nothing is reset (keys of an older epoch read as
// Unknown). The clear-format variant follows.
__global__ void __launch_bounds__(256, VXM_MERGE_MINB) merge_epoch_kernel(KParams p, int rows_per_warp) {
  pdl_wait();  // K3's keys and counters
  const int s = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_merge = global_ns();
  const FrameParams* fp = p.frames + s;
  const uint32_t epoch = fp->epoch;
  const uint32_t cur = fp->cur;
  const int ox = fp->off[0], oy = fp->off[1], oz = fp->off[2];
  const long long base = static_cast<long long>(s) * p.n;
  const uint8_t* occ = p.occ + base;
  const uint32_t* key = p.key + base;
  const uint8_t* src = (cur ? p.loc1 : p.loc0) + base;
  uint8_t* dst = (cur ? p.loc0 : p.loc1) + base;
  const int lane = threadIdx.x & 31;
  const int warp_id = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int rows = p.dy * p.dz;
  const uint32_t dxy = static_cast<uint32_t>(p.dx) * p.dy;

  // packed publish (k4_publish, grids of fewer than 2^24 cells): the block counts
  // travel in one 64-bit atomic with the block count and the last block folds
  // K3's partials itself, so no block waits on a fence except block 0 (its
  // t_merge stamp)
  const bool packed = p.k4_publish && p.n < (1LL << 24) && gridDim.x < 65536u;
  if (!packed && blockIdx.x == 0 && threadIdx.x < 32) fold_trace_slots(p.counters[s]);

  unsigned occ_n = 0, free_n = 0;
  const bool vec = (p.dx & 3) == 0 && (ox & 3) == 0;
  if (ox == 0 && (p.dx & 3) == 0 && p.dx >= 16 && (p.n & 15) == 0 && p.n < (1 << 24)) {
    // No x shift: destination cell c reads c + delta (delta = off_y*dx +
    // off_z*dx*dy), and the valid destination cells of a slab are one run of
    // whole rows. A thread takes 16 consecutive cells: 16 local and occupancy
    // bytes and 16 keys, no per-row arithmetic. A chunk spans at most two
    // rows (dx >= 16), so it is valid throughout when its first and last
    // cells are; chunks at a run boundary test their words one by one (a
    // word never straddles a row since dx % 4 == 0).
    const uint32_t dx = p.dx;
    const int delta = oy * p.dx + oz * static_cast<int>(dxy);
    const int ylo = max(0, -oy), yhi = min(p.dy, p.dy - oy), zlo = max(0, -oz), zhi = min(p.dz, p.dz - oz);
    const float inv_dx = 1.0f / static_cast<float>(dx), inv_dxy = 1.0f / static_cast<float>(dxy);
    auto valid = [&](uint32_t c) {
      const uint32_t z = div_small(c, dxy, inv_dxy);
      const uint32_t y = div_small(c - z * dxy, dx, inv_dx);
      return static_cast<int>(y) >= ylo && static_cast<int>(y) < yhi && static_cast<int>(z) >= zlo &&
             static_cast<int>(z) < zhi;
    };
    const bool aligned = (delta & 15) == 0;
    const uint32_t nch = static_cast<uint32_t>(p.n >> 4);
#if VXM_MERGE_INCR
    // the chunk's (x, y, z) advanced by the grid stride with carries (one
    // division pair for the first chunk and one for the stride) instead of
    // two division pairs per chunk; the chunk's last cell is in the same row
    // or the next one (dx >= 16)
    const uint32_t ch0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    uint32_t cz = div_small(ch0 << 4, dxy, inv_dxy), cy, cx;
    cy = div_small((ch0 << 4) - cz * dxy, dx, inv_dx);
    cx = (ch0 << 4) - cz * dxy - cy * dx;
    const uint32_t S = stride << 4;
    const uint32_t sz = S / dxy, sy = (S - sz * dxy) / dx, sx = S - sz * dxy - sy * dx;
    const int dyi = p.dy;
    for (uint32_t ch = ch0; ch < nch; ch += stride) {
      const uint32_t c = ch << 4;
      const int sc = static_cast<int>(c) + delta;
      uint32_t out[4] = {0u, 0u, 0u, 0u};
      const bool row0 = static_cast<int>(cy) >= ylo && static_cast<int>(cy) < yhi && static_cast<int>(cz) >= zlo &&
                        static_cast<int>(cz) < zhi;
      // the row of cell c + 15
      int ey = static_cast<int>(cy), ez = static_cast<int>(cz);
      if (cx + 15 >= dx) {
        if (++ey == dyi) { ey = 0; ++ez; }
      }
      const bool row1 = ey >= ylo && ey < yhi && ez >= zlo && ez < zhi;
      cx += sx;
      cy += sy;
      cz += sz;
      if (cx >= dx) { cx -= dx; ++cy; }
      if (cy >= static_cast<uint32_t>(dyi)) { cy -= dyi; ++cz; }
      if (row0 && row1) {
#else
    for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nch; ch += gridDim.x * blockDim.x) {
      const uint32_t c = ch << 4;
      const int sc = static_cast<int>(c) + delta;
      uint32_t out[4] = {0u, 0u, 0u, 0u};
      if (valid(c) && valid(c + 15)) {
#endif
        uint32_t l[4], o[4];
        if (aligned) {
          const uint4 L = __ldcs(reinterpret_cast<const uint4*>(src + sc));
          const uint4 O = __ldcs(reinterpret_cast<const uint4*>(occ + sc));
          l[0] = L.x; l[1] = L.y; l[2] = L.z; l[3] = L.w;
          o[0] = O.x; o[1] = O.y; o[2] = O.z; o[3] = O.w;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            l[i] = __ldcs(reinterpret_cast<const unsigned int*>(src + sc + 4 * i));
            o[i] = __ldcs(reinterpret_cast<const unsigned int*>(occ + sc + 4 * i));
          }
        }
        uint4 k[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) k[i] = __ldcs(reinterpret_cast<const uint4*>(key + sc + 4 * i));
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = merge4(l[i], o[i], k[i], epoch);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (valid(c + 4 * i)) {
            const int si = sc + 4 * i;
            out[i] = merge4(*reinterpret_cast<const uint32_t*>(src + si), *reinterpret_cast<const uint32_t*>(occ + si),
                            *reinterpret_cast<const uint4*>(key + si), epoch);
          }
        }
      }
#if VXM_MERGE_STCS
      __stcs(reinterpret_cast<uint4*>(dst + c), make_uint4(out[0], out[1], out[2], out[3]));
#else
      *reinterpret_cast<uint4*>(dst + c) = make_uint4(out[0], out[1], out[2], out[3]);
#endif
      occ_n += count_occupied16(out);
      free_n += count_free16(out);
    }
  } else
  if (vec && p.dx <= 128 && rows_per_warp % kRowsPerWarp == 0) {
    // A row is at most one 4-cell group per lane: issue the loads of
    // kRowsPerWarp rows before resolving any, so each lane keeps
    // kRowsPerWarp x 24 B in flight (the kernel is HBM-latency bound
    // otherwise); a warp takes rows_per_warp / kRowsPerWarp such groups.
    const int x0 = lane * 4, sx = x0 + ox;
    for (int g = 0; g < rows_per_warp; g += kRowsPerWarp) {
    uint32_t l4[kRowsPerWarp], o4[kRowsPerWarp], drow[kRowsPerWarp];
    uint4 k4[kRowsPerWarp];
    bool ok[kRowsPerWarp], in_row[kRowsPerWarp];
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
      const int row = warp_id * rows_per_warp + g + rr;
      const int z = row / p.dy;
      const int y = row - z * p.dy;
      const int sy = y + oy, sz = z + oz;
      in_row[rr] = row < rows && x0 < p.dx;
      ok[rr] = in_row[rr] && sy >= 0 && sy < p.dy && sz >= 0 && sz < p.dz && sx >= 0 && sx < p.dx;
      drow[rr] = static_cast<uint32_t>(y) * p.dx + static_cast<uint32_t>(z) * dxy;
      const long long sc = static_cast<long long>(sy) * p.dx + static_cast<long long>(sz) * dxy + sx;
      l4[rr] = o4[rr] = 0u;
      k4[rr] = make_uint4(0u, 0u, 0u, 0u);
      if (ok[rr]) {
        l4[rr] = __ldcs(reinterpret_cast<const unsigned int*>(src + sc));
        o4[rr] = __ldcs(reinterpret_cast<const unsigned int*>(occ + sc));
        k4[rr] = __ldcs(reinterpret_cast<const uint4*>(key + sc));
      }
    }
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
      if (!in_row[rr]) continue;
      const uint32_t out = ok[rr] ? merge4(l4[rr], o4[rr], k4[rr], epoch) : 0u;
      occ_n += count_occupied4(out);
      free_n += count_free4(out);
      *reinterpret_cast<uint32_t*>(dst + drow[rr] + x0) = out;
    }
    }
  } else
  for (int rr = 0; rr < rows_per_warp; ++rr) {
    const int row = warp_id * rows_per_warp + rr;
    if (row >= rows) break;
    const int z = row / p.dy;
    const int y = row - z * p.dy;
    const int sy = y + oy, sz = z + oz;
    const bool row_ok = sy >= 0 && sy < p.dy && sz >= 0 && sz < p.dz;
    const uint32_t drow = static_cast<uint32_t>(y) * p.dx + static_cast<uint32_t>(z) * dxy;
    const long long srow = static_cast<long long>(sy) * p.dx + static_cast<long long>(sz) * dxy;
    if (vec) {
      for (int x0 = lane * 4; x0 < p.dx; x0 += 128) {
        const int sx = x0 + ox;
        uint32_t out = 0;
        if (row_ok && sx >= 0 && sx < p.dx) {
          const long long sc = srow + sx;
          out = merge4(*reinterpret_cast<const uint32_t*>(src + sc), *reinterpret_cast<const uint32_t*>(occ + sc),
                       *reinterpret_cast<const uint4*>(key + sc), epoch);
        }
        occ_n += count_occupied4(out);
        free_n += count_free4(out);
        *reinterpret_cast<uint32_t*>(dst + drow + x0) = out;
      }
    } else {
      for (int x0 = lane * 4; x0 < p.dx; x0 += 128) {
        for (int i = 0; i < 4 && x0 + i < p.dx; ++i) {
          const int sx = x0 + i + ox;
          uint32_t v = 0;
          if (row_ok && sx >= 0 && sx < p.dx) {
            const long long sc = srow + sx;
            v = merge_cell(src[sc], decode_cell(occ[sc], key[sc], epoch));
          }
          occ_n += v == 2u;
          free_n += v == 1u;
          dst[drow + x0 + i] = static_cast<uint8_t>(v);
        }
      }
    }
  }
  if (packed) {
    publish_packed(p, s, occ_n, free_n);
    return;
  }
  unsigned vals[2] = {occ_n, free_n};
  unsigned long long* dsts[2] = {&p.counters[s].occupied, &p.counters[s].freed};
  block_accumulate<2>(vals, dsts);  // ends after every warp's work (a block barrier)
  if (threadIdx.x == 0) atomicMax(&p.counters[s].t_end, global_ns());
  if (p.k4_publish) publish_when_last(p, s);
}

// Clear-format keys of the source cells the shifted gather never reads
// (their destination lies outside the grid) are reset to Unknown here: x in
// [0, ox) for ox > 0 or [dx + ox, dx) for ox < 0 (every y, z), and likewise
// along y and z (cells in two slabs are written twice). Every other key is
// read, and reset if touched, by the gather itself, so the slot's keys are
// all Unknown again.
__device__ __forceinline__ void clear_orphan_keys(uint32_t* key, int dx, int dy, int dz, int ox, int oy, int oz,
                                                  long long tid, long long nthreads) {
  const int dims[3] = {dx, dy, dz}, off[3] = {ox, oy, oz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int o = off[a], d = dims[a];
    if (o == 0) continue;
    const int lo = o > 0 ? 0 : max(d + o, 0), hi = o > 0 ? min(o, d) : d;
    const long long w = hi - lo;
    // the slab as (x, y, z) with axis a restricted to [lo, hi)
    const long long ex = a == 0 ? w : dx, ey = a == 1 ? w : dy;
    const long long cnt = ex * ey * (a == 2 ? w : dz);
    for (long long i = tid; i < cnt; i += nthreads) {
      const long long x = i % ex, r = i / ex;
      const long long y = r % ey, z = r / ey;
      const long long cx = a == 0 ? lo + x : x, cy = a == 1 ? lo + y : y, cz = a == 2 ? lo + z : z;
      key[cx + cy * dx + cz * static_cast<long long>(dx) * dy] = 0u;
    }
  }
}

// The measurement states of 4 consecutive cells at source cell c (a multiple
// of 4 away from a 16-byte boundary of the key array): epoch format from the
// occupancy bytes and keys; clear format from the keys alone, which are then
// reset to Unknown if the frame touched them.
template <bool kClear>
__device__ __forceinline__ uint32_t meas4(const uint8_t* occ, uint32_t* key, long long c, uint32_t epoch) {
  const uint4 k = __ldcs(reinterpret_cast<const uint4*>(key + c));
  if constexpr (kClear) {
    if (touched4(k)) *reinterpret_cast<uint4*>(key + c) = make_uint4(0u, 0u, 0u, 0u);
    return states4_clear(k);
  } else {
    return states4_epoch(__ldcs(reinterpret_cast<const unsigned int*>(occ + c)), k, epoch);
  }
}
template <bool kClear>
__device__ __forceinline__ uint32_t meas1(const uint8_t* occ, uint32_t* key, long long c, uint32_t epoch) {
  const uint32_t k = key[c];
  if constexpr (kClear) {
    if (k) key[c] = 0u;
    return decode_clear_key(k);
  } else {
    return decode_cell(occ[c], k, epoch);
  }
}

template <bool kClear>
__global__ void __launch_bounds__(256) merge_shift_count_kernel(KParams p, int rows_per_warp) {
  pdl_wait();  // K3's keys and counters
  const int s = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_merge = global_ns();
  const FrameParams* fp = p.frames + s;
  const uint32_t epoch = fp->epoch;
  const uint32_t cur = fp->cur;
  const int ox = fp->off[0], oy = fp->off[1], oz = fp->off[2];
  const long long base = static_cast<long long>(s) * p.n;
  const uint8_t* occ = p.occ + base;
  uint32_t* key = p.key + base;
  const uint8_t* src = (cur ? p.loc1 : p.loc0) + base;
  uint8_t* dst = (cur ? p.loc0 : p.loc1) + base;
  const int lane = threadIdx.x & 31;
  const int warp_id = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int rows = p.dy * p.dz;
  const uint32_t dxy = static_cast<uint32_t>(p.dx) * p.dy;

  if (blockIdx.x == 0 && threadIdx.x < 32) fold_trace_slots(p.counters[s]);

  unsigned occ_n = 0, free_n = 0;
  const bool vec = (p.dx & 3) == 0 && (ox & 3) == 0;
  if (ox == 0 && (p.dx & 3) == 0 && p.dx >= 16 && (p.n & 15) == 0 && p.n < (1 << 24)) {
    // No x shift: destination cell c reads c + delta (delta = off_y*dx +
    // off_z*dx*dy), and the valid destination cells of a slab are one run of
    // whole rows. A thread takes 16 consecutive cells (16 local bytes, their
    // keys and, epoch format, occupancy bytes), no per-row arithmetic. A
    // chunk spans at most two rows (dx >= 16), so it is valid throughout when
    // its first and last cells are; chunks at a run boundary test their words
    // one by one (a word never straddles a row since dx % 4 == 0).
    const uint32_t dx = p.dx;
    const int delta = oy * p.dx + oz * static_cast<int>(dxy);
    const int ylo = max(0, -oy), yhi = min(p.dy, p.dy - oy), zlo = max(0, -oz), zhi = min(p.dz, p.dz - oz);
    const float inv_dx = 1.0f / static_cast<float>(dx), inv_dxy = 1.0f / static_cast<float>(dxy);
    auto valid = [&](uint32_t c) {
      const uint32_t z = div_small(c, dxy, inv_dxy);
      const uint32_t y = div_small(c - z * dxy, dx, inv_dx);
      return static_cast<int>(y) >= ylo && static_cast<int>(y) < yhi && static_cast<int>(z) >= zlo &&
             static_cast<int>(z) < zhi;
    };
    const bool aligned = (delta & 15) == 0;
    const uint32_t nch = static_cast<uint32_t>(p.n >> 4);
    for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nch; ch += gridDim.x * blockDim.x) {
      const uint32_t c = ch << 4;
      const int sc = static_cast<int>(c) + delta;
      uint32_t out[4] = {0u, 0u, 0u, 0u};
      if (valid(c) && valid(c + 15)) {
        uint32_t l[4], o[4] = {0u, 0u, 0u, 0u};
        if (aligned) {
          const uint4 L = __ldcs(reinterpret_cast<const uint4*>(src + sc));
          l[0] = L.x; l[1] = L.y; l[2] = L.z; l[3] = L.w;
          if constexpr (!kClear) {
            const uint4 O = __ldcs(reinterpret_cast<const uint4*>(occ + sc));
            o[0] = O.x; o[1] = O.y; o[2] = O.z; o[3] = O.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            l[i] = __ldcs(reinterpret_cast<const unsigned int*>(src + sc + 4 * i));
            if constexpr (!kClear) o[i] = __ldcs(reinterpret_cast<const unsigned int*>(occ + sc + 4 * i));
          }
        }
        uint4 k[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) k[i] = __ldcs(reinterpret_cast<const uint4*>(key + sc + 4 * i));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if constexpr (kClear) {
            out[i] = merge4s(l[i], states4_clear(k[i]));
            if (touched4(k[i])) *reinterpret_cast<uint4*>(key + sc + 4 * i) = make_uint4(0u, 0u, 0u, 0u);
          } else {
            out[i] = merge4s(l[i], states4_epoch(o[i], k[i], epoch));
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (valid(c + 4 * i)) {
            const int si = sc + 4 * i;
            out[i] = merge4s(*reinterpret_cast<const uint32_t*>(src + si), meas4<kClear>(occ, key, si, epoch));
          }
        }
      }
#if VXM_MERGE_STCS
      __stcs(reinterpret_cast<uint4*>(dst + c), make_uint4(out[0], out[1], out[2], out[3]));
#else
      *reinterpret_cast<uint4*>(dst + c) = make_uint4(out[0], out[1], out[2], out[3]);
#endif
      occ_n += count_occupied16(out);
      free_n += count_free16(out);
    }
  } else
  if (vec && p.dx <= 128 && rows_per_warp == kRowsPerWarp) {
    // A row is at most one 4-cell group per lane: issue the loads of all the
    // warp's rows before resolving any, so each lane keeps kRowsPerWarp x 24 B
    // in flight (the kernel is HBM-latency bound otherwise).
    const int x0 = lane * 4, sx = x0 + ox;
    uint32_t l4[kRowsPerWarp], o4[kRowsPerWarp], drow[kRowsPerWarp];
    long long scell[kRowsPerWarp];
    uint4 k4[kRowsPerWarp];
    bool ok[kRowsPerWarp], in_row[kRowsPerWarp];
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
      const int row = warp_id * kRowsPerWarp + rr;
      const int z = row / p.dy;
      const int y = row - z * p.dy;
      const int sy = y + oy, sz = z + oz;
      in_row[rr] = row < rows && x0 < p.dx;
      ok[rr] = in_row[rr] && sy >= 0 && sy < p.dy && sz >= 0 && sz < p.dz && sx >= 0 && sx < p.dx;
      drow[rr] = static_cast<uint32_t>(y) * p.dx + static_cast<uint32_t>(z) * dxy;
      const long long sc = static_cast<long long>(sy) * p.dx + static_cast<long long>(sz) * dxy + sx;
      scell[rr] = sc;
      l4[rr] = o4[rr] = 0u;
      k4[rr] = make_uint4(0u, 0u, 0u, 0u);
      if (ok[rr]) {
        l4[rr] = __ldcs(reinterpret_cast<const unsigned int*>(src + sc));
        if constexpr (!kClear) o4[rr] = __ldcs(reinterpret_cast<const unsigned int*>(occ + sc));
        k4[rr] = __ldcs(reinterpret_cast<const uint4*>(key + sc));
      }
    }
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
      if (!in_row[rr]) continue;
      uint32_t out = 0u;
      if (ok[rr]) {
        if constexpr (kClear) {
          out = merge4s(l4[rr], states4_clear(k4[rr]));
          if (touched4(k4[rr])) *reinterpret_cast<uint4*>(key + scell[rr]) = make_uint4(0u, 0u, 0u, 0u);
        } else {
          out = merge4s(l4[rr], states4_epoch(o4[rr], k4[rr], epoch));
        }
      }
      occ_n += count_occupied4(out);
      free_n += count_free4(out);
      *reinterpret_cast<uint32_t*>(dst + drow[rr] + x0) = out;
    }
  } else
  for (int rr = 0; rr < rows_per_warp; ++rr) {
    const int row = warp_id * rows_per_warp + rr;
    if (row >= rows) break;
    const int z = row / p.dy;
    const int y = row - z * p.dy;
    const int sy = y + oy, sz = z + oz;
    const bool row_ok = sy >= 0 && sy < p.dy && sz >= 0 && sz < p.dz;
    const uint32_t drow = static_cast<uint32_t>(y) * p.dx + static_cast<uint32_t>(z) * dxy;
    const long long srow = static_cast<long long>(sy) * p.dx + static_cast<long long>(sz) * dxy;
    if (vec) {
      for (int x0 = lane * 4; x0 < p.dx; x0 += 128) {
        const int sx = x0 + ox;
        uint32_t out = 0;
        if (row_ok && sx >= 0 && sx < p.dx) {
          const long long sc = srow + sx;
          out = merge4s(*reinterpret_cast<const uint32_t*>(src + sc), meas4<kClear>(occ, key, sc, epoch));
        }
        occ_n += count_occupied4(out);
        free_n += count_free4(out);
        *reinterpret_cast<uint32_t*>(dst + drow + x0) = out;
      }
    } else {
      for (int x0 = lane * 4; x0 < p.dx; x0 += 128) {
        for (int i = 0; i < 4 && x0 + i < p.dx; ++i) {
          const int sx = x0 + i + ox;
          uint32_t v = 0;
          if (row_ok && sx >= 0 && sx < p.dx) {
            const long long sc = srow + sx;
            v = merge_cell(src[sc], meas1<kClear>(occ, key, sc, epoch));
          }
          occ_n += v == 2u;
          free_n += v == 1u;
          dst[drow + x0 + i] = static_cast<uint8_t>(v);
        }
      }
    }
  }
  if constexpr (kClear)
    clear_orphan_keys(key, p.dx, p.dy, p.dz, ox, oy, oz, static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x,
                      static_cast<long long>(gridDim.x) * blockDim.x);
  unsigned vals[2] = {occ_n, free_n};
  unsigned long long* dsts[2] = {&p.counters[s].occupied, &p.counters[s].freed};
  block_accumulate<2>(vals, dsts);  // ends after every warp's work (a block barrier)
  if (threadIdx.x == 0) atomicMax(&p.counters[s].t_end, global_ns());
}


// K4, TMA-staged: a group is merge_tma_rows(dx, dy) consecutive x-rows of
// one z-slab (about kMergeStageCells cells, so one stage is ~19 KB whatever
// the row length); each block pipelines several groups through two stages.
// The source rows these come from after the shift (rows y + off_y of slab
// z + off_z) are contiguous in memory, so one elected thread stages them with
// bulk copies (local bytes, keys and, epoch format, occupancy bytes; each
// window widened to 16-byte boundaries) on one mbarrier, and the warps merge,
// shift and count out of shared memory: 4 cells per lane as one word when
// dims_x and the x shift are multiples of 4, else cell by cell (clear-format
// keys the frame touched are reset in global memory as they are consumed).
// Needs 16 bytes of slack after each array (allocated by the runtime).
constexpr int kMergeStageCells = 3200;
constexpr int kMergeTmaMaxDx = 1024;  // larger rows take the direct-load K4

__host__ __device__ constexpr int merge_tma_rows(int dx, int dy) {
  return kMergeStageCells / dx < 1 ? 1 : (kMergeStageCells / dx < dy ? kMergeStageCells / dx : dy);
}
// one stage: local and occupancy bytes and keys of `cells` cells, each
// window widened to 16-byte boundaries
__host__ __device__ constexpr size_t merge_tma_smem_bytes(int cells) {
  // rounded to 16 bytes: the second stage starts right after the first and
  // bulk copies need 16-byte aligned destinations
  return (2 * (static_cast<size_t>(cells) + 32) + 4 * static_cast<size_t>(cells) + 32 + 15) & ~static_cast<size_t>(15);
}

__device__ __forceinline__ const unsigned char* align16_down(const void* p) {
  return reinterpret_cast<const unsigned char*>(reinterpret_cast<uintptr_t>(p) & ~static_cast<uintptr_t>(15));
}
__device__ __forceinline__ const unsigned char* align16_up(const void* p) {
  return reinterpret_cast<const unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~static_cast<uintptr_t>(15));
}

__global__ void __launch_bounds__(256) merge_epoch_tma_kernel(KParams p) {
  extern __shared__ __align__(16) unsigned char msm[];
  __shared__ uint64_t bar[2];
  const int s = blockIdx.y;
  const FrameParams* fp = p.frames + s;
  const int dx = p.dx, dy = p.dy, dz = p.dz;
  const long long dxy = static_cast<long long>(dx) * dy;
  const int ox = fp->off[0], oy = fp->off[1], oz = fp->off[2];
  const uint32_t epoch = fp->epoch;
  const uint32_t cur = fp->cur;
  const long long base = static_cast<long long>(s) * p.n;
  const uint8_t* src = (cur ? p.loc1 : p.loc0) + base;
  uint8_t* dst = (cur ? p.loc0 : p.loc1) + base;
  const uint8_t* occ = p.occ + base;
  const uint32_t* key = p.key + base;
  const int rows = merge_tma_rows(dx, dy);
  const int ngy = (dy + rows - 1) / rows;
  const int ngroups = ngy * dz;
  const size_t stage_bytes = merge_tma_smem_bytes(rows * dx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = ((dx | ox) & 3) == 0;

  // geometry of group g: rows [y0, y0 + ny) of slab z, sourced from rows
  // [sy_lo, sy_hi) of slab z + off_z (cells [c0, c1) of the slot)
  struct Group {
    int y0, ny, z, sy_lo, sy_hi;
    bool any;
    long long c0, c1;
  };
  auto group = [&](int g) {
    Group G;
    G.z = g / ngy;
    G.y0 = (g - G.z * ngy) * rows;
    G.ny = min(rows, dy - G.y0);
    const int sz = G.z + oz;
    G.sy_lo = max(0, G.y0 + oy);
    G.sy_hi = min(dy, G.y0 + oy + G.ny);
    G.any = sz >= 0 && sz < dz && G.sy_lo < G.sy_hi;
    G.c0 = static_cast<long long>(G.sy_lo) * dx + sz * dxy;
    G.c1 = static_cast<long long>(G.sy_hi) * dx + sz * dxy;
    return G;
  };
  // one elected thread stages group g into stage buffer b (possibly nothing)
  auto issue = [&](int g, int b) {
    const Group G = group(g);
    unsigned char* sl = msm + b * stage_bytes;
    uint32_t lb = 0, ob = 0, kb = 0;
    const unsigned char *lw0 = nullptr, *ow0 = nullptr, *kw0 = nullptr;
    if (G.any) {
      lw0 = align16_down(src + G.c0);
      ow0 = align16_down(occ + G.c0);
      kw0 = align16_down(key + G.c0);
      lb = static_cast<uint32_t>(align16_up(src + G.c1) - lw0);
      ob = static_cast<uint32_t>(align16_up(occ + G.c1) - ow0);
      kb = static_cast<uint32_t>(align16_up(key + G.c1) - kw0);
    }
    mbar_expect_tx(&bar[b], lb + ob + kb);
    if (G.any) {
      unsigned char* so = sl + ((lb + 15u) & ~15u);
      unsigned char* sk = so + ((ob + 15u) & ~15u);
      bulk_g2s(sl, lw0, lb, &bar[b]);
      bulk_g2s(so, ow0, ob, &bar[b]);
      bulk_g2s(sk, kw0, kb, &bar[b]);
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // K3's keys and counters
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_merge = global_ns();
  if (blockIdx.x == 0 && threadIdx.x < 32) fold_trace_slots(p.counters[s]);
  unsigned occ_n = 0, free_n = 0;
  int g = blockIdx.x;
  if (g < ngroups && threadIdx.x == 0) issue(g, 0);
  for (int it = 0; g < ngroups; ++it, g += gridDim.x) {
    const int b = it & 1;
    // refill the other stage (consumed in the previous iteration, after its
    // closing barrier) while this one lands
    if (g + gridDim.x < ngroups && threadIdx.x == 0) issue(g + gridDim.x, b ^ 1);
    mbar_wait(&bar[b], (it >> 1) & 1);
    const Group G = group(g);
    const unsigned char* sl = msm + b * stage_bytes;
    int ll = 0, ol = 0, kl = 0;
    const unsigned char *so = sl, *sk = sl;
    if (G.any) {
      const unsigned char* lw0 = align16_down(src + G.c0);
      const unsigned char* ow0 = align16_down(occ + G.c0);
      const unsigned char* kw0 = align16_down(key + G.c0);
      const uint32_t lb = static_cast<uint32_t>(align16_up(src + G.c1) - lw0);
      const uint32_t ob = static_cast<uint32_t>(align16_up(occ + G.c1) - ow0);
      so = sl + ((lb + 15u) & ~15u);
      sk = so + ((ob + 15u) & ~15u);
      ll = static_cast<int>((src + G.c0) - lw0);
      ol = static_cast<int>((occ + G.c0) - ow0);
      kl = static_cast<int>(reinterpret_cast<const unsigned char*>(key + G.c0) - kw0);
    }
    for (int r = warp; r < G.ny; r += blockDim.x >> 5) {
      const int y = G.y0 + r, sy = y + oy;
      const bool row_ok = G.any && sy >= G.sy_lo && sy < G.sy_hi;
      uint8_t* drow = dst + static_cast<long long>(y) * dx + G.z * dxy;
      const long long rrow = static_cast<long long>(sy - G.sy_lo) * dx;  // relative to c0
      for (int x0 = lane * 4; x0 < dx; x0 += 128) {
        uint32_t out = 0;
        if (vec) {
          const int sx = x0 + ox;
          if (row_ok && sx >= 0 && sx < dx) {
            const long long rel = rrow + sx;
            out = merge4(*reinterpret_cast<const uint32_t*>(sl + ll + rel),
                         *reinterpret_cast<const uint32_t*>(so + ol + rel),
                         *reinterpret_cast<const uint4*>(sk + kl + 4 * rel), epoch);
          }
          *reinterpret_cast<uint32_t*>(drow + x0) = out;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int x = x0 + k, sx = x + ox;
            if (x >= dx) break;
            uint32_t v = 0;
            if (row_ok && sx >= 0 && sx < dx) {
              const long long rel = rrow + sx;
              v = merge_cell(sl[ll + rel],
                             decode_cell(so[ol + rel], *reinterpret_cast<const uint32_t*>(sk + kl + 4 * rel), epoch));
            }
            out |= v << (8 * k);
            drow[x] = static_cast<uint8_t>(v);
          }
        }
        occ_n += count_occupied4(out);
        free_n += count_free4(out);
      }
    }
    __syncthreads();  // stage b is refilled two groups from now
  }
  // every warp has passed the last group's barrier
  if (threadIdx.x == 0) atomicMax(&p.counters[s].t_end, global_ns());
  unsigned vals[2] = {occ_n, free_n};
  unsigned long long* dsts[2] = {&p.counters[s].occupied, &p.counters[s].freed};
  warp_accumulate<2>(vals, dsts);
}

template <bool kClear>
__global__ void __launch_bounds__(256) merge_shift_count_tma_kernel(KParams p) {
  extern __shared__ __align__(16) unsigned char msm[];
  __shared__ uint64_t bar[2];
  const int s = blockIdx.y;
  const FrameParams* fp = p.frames + s;
  const int dx = p.dx, dy = p.dy, dz = p.dz;
  const long long dxy = static_cast<long long>(dx) * dy;
  const int ox = fp->off[0], oy = fp->off[1], oz = fp->off[2];
  const uint32_t epoch = fp->epoch;
  const uint32_t cur = fp->cur;
  const long long base = static_cast<long long>(s) * p.n;
  const uint8_t* src = (cur ? p.loc1 : p.loc0) + base;
  uint8_t* dst = (cur ? p.loc0 : p.loc1) + base;
  const uint8_t* occ = p.occ + base;
  uint32_t* key = p.key + base;
  const int rows = merge_tma_rows(dx, dy);
  const int ngy = (dy + rows - 1) / rows;
  const int ngroups = ngy * dz;
  const size_t stage_bytes = merge_tma_smem_bytes(rows * dx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = ((dx | ox) & 3) == 0;

  // geometry of group g: rows [y0, y0 + ny) of slab z, sourced from rows
  // [sy_lo, sy_hi) of slab z + off_z (cells [c0, c1) of the slot)
  struct Group {
    int y0, ny, z, sy_lo, sy_hi;
    bool any;
    long long c0, c1;
  };
  auto group = [&](int g) {
    Group G;
    G.z = g / ngy;
    G.y0 = (g - G.z * ngy) * rows;
    G.ny = min(rows, dy - G.y0);
    const int sz = G.z + oz;
    G.sy_lo = max(0, G.y0 + oy);
    G.sy_hi = min(dy, G.y0 + oy + G.ny);
    G.any = sz >= 0 && sz < dz && G.sy_lo < G.sy_hi;
    G.c0 = static_cast<long long>(G.sy_lo) * dx + sz * dxy;
    G.c1 = static_cast<long long>(G.sy_hi) * dx + sz * dxy;
    return G;
  };
  // one elected thread stages group g into stage buffer b (possibly nothing)
  auto issue = [&](int g, int b) {
    const Group G = group(g);
    unsigned char* sl = msm + b * stage_bytes;
    uint32_t lb = 0, ob = 0, kb = 0;
    const unsigned char *lw0 = nullptr, *ow0 = nullptr, *kw0 = nullptr;
    if (G.any) {
      lw0 = align16_down(src + G.c0);
      kw0 = align16_down(key + G.c0);
      lb = static_cast<uint32_t>(align16_up(src + G.c1) - lw0);
      kb = static_cast<uint32_t>(align16_up(key + G.c1) - kw0);
      if constexpr (!kClear) {
        ow0 = align16_down(occ + G.c0);
        ob = static_cast<uint32_t>(align16_up(occ + G.c1) - ow0);
      }
    }
    mbar_expect_tx(&bar[b], lb + ob + kb);
    if (G.any) {
      unsigned char* so = sl + ((lb + 15u) & ~15u);
      unsigned char* sk = so + ((ob + 15u) & ~15u);
      bulk_g2s(sl, lw0, lb, &bar[b]);
      if constexpr (!kClear) bulk_g2s(so, ow0, ob, &bar[b]);
      bulk_g2s(sk, kw0, kb, &bar[b]);
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // K3's keys and counters
  if (blockIdx.x == 0 && threadIdx.x == 0) p.counters[s].t_merge = global_ns();
  if (blockIdx.x == 0 && threadIdx.x < 32) fold_trace_slots(p.counters[s]);
  unsigned occ_n = 0, free_n = 0;
  int g = blockIdx.x;
  if (g < ngroups && threadIdx.x == 0) issue(g, 0);
  for (int it = 0; g < ngroups; ++it, g += gridDim.x) {
    const int b = it & 1;
    // refill the other stage (consumed in the previous iteration, after its
    // closing barrier) while this one lands
    if (g + gridDim.x < ngroups && threadIdx.x == 0) issue(g + gridDim.x, b ^ 1);
    mbar_wait(&bar[b], (it >> 1) & 1);
    const Group G = group(g);
    const unsigned char* sl = msm + b * stage_bytes;
    int ll = 0, ol = 0, kl = 0;
    const unsigned char *so = sl, *sk = sl;
    if (G.any) {
      const unsigned char* lw0 = align16_down(src + G.c0);
      const unsigned char* kw0 = align16_down(key + G.c0);
      const uint32_t lb = static_cast<uint32_t>(align16_up(src + G.c1) - lw0);
      uint32_t ob = 0;
      so = sl + ((lb + 15u) & ~15u);
      if constexpr (!kClear) {
        const unsigned char* ow0 = align16_down(occ + G.c0);
        ob = static_cast<uint32_t>(align16_up(occ + G.c1) - ow0);
        ol = static_cast<int>((occ + G.c0) - ow0);
      }
      sk = so + ((ob + 15u) & ~15u);
      ll = static_cast<int>((src + G.c0) - lw0);
      kl = static_cast<int>(reinterpret_cast<const unsigned char*>(key + G.c0) - kw0);
    }
    uint32_t* const kg = key + G.c0;  // the group's keys in global memory (clear format: reset there)
    for (int r = warp; r < G.ny; r += blockDim.x >> 5) {
      const int y = G.y0 + r, sy = y + oy;
      const bool row_ok = G.any && sy >= G.sy_lo && sy < G.sy_hi;
      uint8_t* drow = dst + static_cast<long long>(y) * dx + G.z * dxy;
      const long long rrow = static_cast<long long>(sy - G.sy_lo) * dx;  // relative to c0
      for (int x0 = lane * 4; x0 < dx; x0 += 128) {
        uint32_t out = 0;
        if (vec) {
          const int sx = x0 + ox;
          if (row_ok && sx >= 0 && sx < dx) {
            const long long rel = rrow + sx;
            const uint4 k = *reinterpret_cast<const uint4*>(sk + kl + 4 * rel);
            uint32_t m4;
            if constexpr (kClear) {
              m4 = states4_clear(k);
              if (touched4(k)) *reinterpret_cast<uint4*>(kg + rel) = make_uint4(0u, 0u, 0u, 0u);
            } else {
              m4 = states4_epoch(*reinterpret_cast<const uint32_t*>(so + ol + rel), k, epoch);
            }
            out = merge4s(*reinterpret_cast<const uint32_t*>(sl + ll + rel), m4);
          }
          *reinterpret_cast<uint32_t*>(drow + x0) = out;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int x = x0 + k, sx = x + ox;
            if (x >= dx) break;
            uint32_t v = 0;
            if (row_ok && sx >= 0 && sx < dx) {
              const long long rel = rrow + sx;
              const uint32_t kk = *reinterpret_cast<const uint32_t*>(sk + kl + 4 * rel);
              uint32_t m;
              if constexpr (kClear) {
                m = decode_clear_key(kk);
                if (kk) kg[rel] = 0u;
              } else {
                m = decode_cell(so[ol + rel], kk, epoch);
              }
              v = merge_cell(sl[ll + rel], m);
            }
            out |= v << (8 * k);
            drow[x] = static_cast<uint8_t>(v);
          }
        }
        occ_n += count_occupied4(out);
        free_n += count_free4(out);
      }
    }
    __syncthreads();  // stage b is refilled two groups from now
  }
  if constexpr (kClear)
    clear_orphan_keys(key, dx, dy, dz, ox, oy, oz, static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x,
                      static_cast<long long>(gridDim.x) * blockDim.x);
  // every warp has passed the last group's barrier
  if (threadIdx.x == 0) atomicMax(&p.counters[s].t_end, global_ns());
  unsigned vals[2] = {occ_n, free_n};
  unsigned long long* dsts[2] = {&p.counters[s].occupied, &p.counters[s].freed};
  warp_accumulate<2>(vals, dsts);
}

// ---------------------------------------------------------------------------
// K4 for F > 1 consecutive frames of each stream in one call (SURVEY §8f
// "next" #1: populate and trace of all F frames run as F independent slots,
// only the merge + shift is a chain). Frame k merges its measurement grid
// into the local grid and then shifts it by off_k (pipeline.cpp:99-112), so
// the value that ends at cell c_k after frame k came from c_{k-1} = c_k +
// off_k: along such a chain g = c_k + P_k (P_k = off_0 + ... + off_k,
// P_{-1} = 0) is invariant. Every (frame, cell) lies on exactly one chain, so
// one thread per chain folds the F merges in order, exactly as F K4 launches
// would, without materialising the intermediate grids:
//   v_k(c_k) = inb(c_{k-1}) ? merge(v_{k-1}(c_{k-1}), ms_k(c_{k-1})) : Unknown
// and counts Occupied / Free of every intermediate grid (the per-frame
// PipelineStats counts, pipeline.cpp:114-115). The chains of a stream span
// the box [min P, max P + dims) (host-computed, FrameParams::box_*); a
// grid-stride loop covers it, so the captured launch shape never changes.
// ---------------------------------------------------------------------------
constexpr int kMaxFramesPerCall = 64;

// Warp sums of per-frame Occupied / Free counts packed as bytes (frame k0+u:
// byte pair u&1 of word u>>1; every warp sum is <= 128), accumulated by the
// lane of each frame and added into the block's per-frame counters (32-bit
// shared atomics: [k] occupied, [kMaxFramesPerCall + k] freed) at the end.
template <int U>
__device__ __forceinline__ void add_frame_counts(const uint32_t (&packed)[U / 2], uint32_t (&acc)[4], int k0, int lane) {
  // Each warp sum lands in the lane of its frame (lane k & 31, frames k and
  // k + 1 of a pair share a half of the 64), flushed once per thread by
  // flush_frame_counts instead of shared atomics every group.
#pragma unroll
  for (int h = 0; h < U / 2; ++h) {
    const uint32_t sum = __reduce_add_sync(0xffffffffu, packed[h]);
    const int fk = k0 + 2 * h;  // even: fk and fk + 1 in the same half
    const uint32_t mine = lane == (fk & 31) ? sum : (lane == ((fk + 1) & 31) ? sum >> 16 : 0u);
    if (fk < 32) {
      acc[0] += mine & 0xffu;
      acc[1] += (mine >> 8) & 0xffu;
    } else {
      acc[2] += mine & 0xffu;
      acc[3] += (mine >> 8) & 0xffu;
    }
  }
}

// the lane accumulators of add_frame_counts into the block's shared counts
__device__ __forceinline__ void flush_frame_counts(const uint32_t (&acc)[4], unsigned* cnt, int lane) {
  if (acc[0]) atomicAdd(&cnt[lane], acc[0]);
  if (acc[1]) atomicAdd(&cnt[kMaxFramesPerCall + lane], acc[1]);
  if (acc[2]) atomicAdd(&cnt[32 + lane], acc[2]);
  if (acc[3]) atomicAdd(&cnt[kMaxFramesPerCall + 32 + lane], acc[3]);
}

// End of a chain-merge block (k4_publish): the stream's last participating
// block (block 0 and every block that did not leave early) publishes its F
// frame slots, one warp per slot, so no K5 follows on the chain of ranges.
// Threadfence reduction: each thread's counter atomics are fenced before the
// block's arrival on merge_done of the stream's first slot.
__device__ __forceinline__ void chain_publish_when_last(const KParams& p, int s, int F, long long work) {
  __shared__ unsigned last;
  const long long nact = max(1LL, min(static_cast<long long>(gridDim.x), (work + blockDim.x - 1) / blockDim.x));
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    last = atomicAdd(&p.counters[static_cast<long long>(s) * F].merge_done, 1ull) ==
                   static_cast<unsigned long long>(nact - 1) ? 1u : 0u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = threadIdx.x >> 5; k < F; k += blockDim.x >> 5)
    publish_slot(p, s * F + k, threadIdx.x & 31, 32);
}

// Warp 0 of a chain-merge block: the cumulative shifts P_{k-1} of the F
// frames (Pc[k], Pc[0] = 0; entries past F repeat P_{F-1}) and their epochs,
// two frames per lane and one warp scan instead of a serial loop over F in
// one thread; *vec_ok = every x shift (and dims_x) is a multiple of 4.
__device__ __forceinline__ void chain_prefix(const FrameParams* f0, int F, int dx, int (*Pc)[3], uint32_t* ep,
                                             int* vec_ok, int lane) {
  static_assert(kMaxFramesPerCall <= 64, "two frames per lane");
  const int k = 2 * lane;
  int a0[3] = {0, 0, 0}, a1[3] = {0, 0, 0}, t[3];
  if (k < F) {
    for (int a = 0; a < 3; ++a) a0[a] = f0[k].off[a];
    ep[k] = f0[k].epoch;
  }
  if (k + 1 < F) {
    for (int a = 0; a < 3; ++a) a1[a] = f0[k + 1].off[a];
    ep[k + 1] = f0[k + 1].epoch;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    t[a] = a0[a] + a1[a];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, t[a], d);
      if (lane >= d) t[a] += v;
    }
    Pc[k + 1][a] = t[a] - a1[a];  // P_k
    Pc[k + 2][a] = t[a];          // P_{k+1}
  }
  if (lane == 0) Pc[0][0] = Pc[0][1] = Pc[0][2] = 0;
  const bool aligned = __all_sync(0xffffffffu, ((t[0] - a1[0]) & 3) == 0 && (t[0] & 3) == 0);
  if (lane == 0) *vec_ok = aligned && (dx & 3) == 0 ? 1 : 0;
}

__global__ void __launch_bounds__(VXM_SEQ_THREADS, VXM_SEQ_MINB * 256 / VXM_SEQ_THREADS) merge_sequence_epoch_kernel(KParams p, int F) {
  pdl_wait();  // K3's keys and counters
  constexpr int U = VXM_SEQ_U;  // frames whose loads are issued together
  __shared__ unsigned cnt[2 * kMaxFramesPerCall];           // occupied, then freed, per frame
  __shared__ int Pc[kMaxFramesPerCall + U][3];              // P_{k-1} at index k
  __shared__ uint32_t ep[kMaxFramesPerCall];
  const int s = blockIdx.y;  // stream
  const FrameParams* f0 = p.frames + static_cast<long long>(s) * F;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0) {
    const unsigned long long t = global_ns();
    for (int k = threadIdx.x; k < F; k += blockDim.x) p.counters[static_cast<long long>(s) * F + k].t_merge = t;
  }
  for (int k = threadIdx.x; k < 2 * kMaxFramesPerCall; k += blockDim.x) cnt[k] = 0u;
  __shared__ int vec_ok;
  if (threadIdx.x < 32) chain_prefix(f0, F, p.dx, Pc, ep, &vec_ok, lane);
  if (blockIdx.x == 0) {
    // fold the trace counters of every frame slot of this stream (one warp each)
    for (int k = threadIdx.x >> 5; k < F; k += blockDim.x >> 5) fold_trace_slots(p.counters[static_cast<long long>(s) * F + k]);
  }
  __syncthreads();
  const int dx = p.dx, dy = p.dy, dz = p.dz;
  const uint32_t dxy = static_cast<uint32_t>(dx) * static_cast<uint32_t>(dy);  // (cells < 2^32)
  const int bx = f0->box_lo[0], by = f0->box_lo[1], bz = f0->box_lo[2];
  const int ex = f0->box_ext[0], ey = f0->box_ext[1], ez = f0->box_ext[2];
  const long long nchain = static_cast<long long>(ex) * ey * ez;
  // blocks past the work (the grid is sized for the largest box) leave
  // before the counters: no idle t_end atomics on the frame slots
  if (blockIdx.x > 0 && static_cast<long long>(blockIdx.x) * blockDim.x >= (vec_ok ? (nchain >> 2) : nchain)) return;
  const uint32_t cur = f0->cur;
  const uint8_t* src = (cur ? p.loc1 : p.loc0) + static_cast<long long>(s) * p.n;
  uint8_t* dst = (cur ? p.loc0 : p.loc1) + static_cast<long long>(s) * p.n;
  const uint8_t* occ0 = p.occ + static_cast<long long>(s) * F * p.n;
  const uint32_t* key0 = p.key + static_cast<long long>(s) * F * p.n;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  uint32_t acc[4] = {0u, 0u, 0u, 0u};  // per-frame Occupied / Free counts, see add_frame_counts
  if (vec_ok) {
    // Every frame's x shift is a multiple of 4 (and dims_x too): a thread
    // folds 4 neighbouring chains at once, moving the 4 cells as one word
    // (occupancy u32, keys uint4) and merging / counting them with the
    // byte-SIMD helpers of K4.
    const int ex4 = ex >> 2;
    const long long ngroup = static_cast<long long>(ex4) * ey * ez;
    for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x; base < ngroup; base += stride) {
      const long long i = base + threadIdx.x;
      const bool active = i < ngroup;
      const int iz = static_cast<int>(i / (static_cast<long long>(ex4) * ey));
      const int rem = static_cast<int>(i - static_cast<long long>(iz) * ex4 * ey);
      const int iy = rem / ex4;
      const int gx = bx + 4 * (rem - iy * ex4), gy = by + iy, gz = bz + iz;
      auto group_of = [&](int k, bool& in) -> uint32_t {  // first cell of the group at c_{k-1}
        const int cx = gx - Pc[k][0], cy = gy - Pc[k][1], cz = gz - Pc[k][2];
        in = active && static_cast<unsigned>(cx) < static_cast<unsigned>(dx) &&
             static_cast<unsigned>(cy) < static_cast<unsigned>(dy) && static_cast<unsigned>(cz) < static_cast<unsigned>(dz);
        return static_cast<uint32_t>(cx) + static_cast<uint32_t>(cy) * static_cast<uint32_t>(dx) +
               static_cast<uint32_t>(cz) * dxy;
      };
      bool in_prev;
      uint32_t pos_prev = group_of(0, in_prev);
      uint32_t val = in_prev ? *reinterpret_cast<const uint32_t*>(src + pos_prev) : 0u;
      auto og = occ0;  // slabs of frame k0 (advanced one frame per load pair)
      auto kg = key0;
      for (int k0 = 0; k0 < F; k0 += U) {
        bool in_c[U];
        uint32_t pos[U];
        uint32_t o[U];
        uint4 kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) pos[u] = group_of(k0 + u + 1, in_c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool in_r = u == 0 ? in_prev : in_c[u - 1];
          const uint32_t r = u == 0 ? pos_prev : pos[u - 1];
          const bool ld = k0 + u < F && in_c[u] && in_r;
          const auto oa = og + r;
          const auto ka = kg + r;
          og += p.n;
          kg += p.n;
          o[u] = ld ? __ldcs(reinterpret_cast<const uint32_t*>(oa)) : 0u;
          kk[u] = ld ? __ldcs(reinterpret_cast<const uint4*>(ka)) : make_uint4(0u, 0u, 0u, 0u);
        }
        // per frame: Occupied / Free counts of this thread's 4 cells (each
        // <= 4, so a warp sum fits a byte); two frames share one reduction
        uint32_t packed[U / 2] = {};
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u;
          if (k >= F) break;
          const bool in_r = u == 0 ? in_prev : in_c[u - 1];
          if (in_c[u]) val = in_r ? merge4(val, o[u], kk[u], ep[k]) : 0u;  // shifted in: Unknown
          const unsigned oc = in_c[u] ? count_occupied4(val) : 0u, fr = in_c[u] ? count_free4(val) : 0u;
          packed[u >> 1] |= (oc | (fr << 8)) << (16 * (u & 1));
        }
        add_frame_counts<U>(packed, acc, k0, lane);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (k0 + u < F) {
            in_prev = in_c[u];
            pos_prev = pos[u];
          }
        }
      }
      if (in_prev) *reinterpret_cast<uint32_t*>(dst + pos_prev) = val;
    }
  } else
  for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x; base < nchain; base += stride) {
    const long long i = base + threadIdx.x;
    const bool active = i < nchain;
    const int iz = static_cast<int>(i / (static_cast<long long>(ex) * ey));
    const int rem = static_cast<int>(i - static_cast<long long>(iz) * ex * ey);
    const int iy = rem / ex;
    const int gx = bx + rem - iy * ex, gy = by + iy, gz = bz + iz;
    auto cell_of = [&](int k, bool& in) -> uint32_t {  // c_{k-1} = g - P_{k-1}
      const int cx = gx - Pc[k][0], cy = gy - Pc[k][1], cz = gz - Pc[k][2];
      in = active && static_cast<unsigned>(cx) < static_cast<unsigned>(dx) &&
           static_cast<unsigned>(cy) < static_cast<unsigned>(dy) && static_cast<unsigned>(cz) < static_cast<unsigned>(dz);
      return static_cast<uint32_t>(cx) + static_cast<uint32_t>(cy) * static_cast<uint32_t>(dx) +
               static_cast<uint32_t>(cz) * dxy;
    };
    bool in_prev;
    uint32_t pos_prev = cell_of(0, in_prev);
    uint32_t val = in_prev ? src[pos_prev] : 0u;
    auto og = occ0;  // slabs of frame k0 (advanced one frame per load pair)
    auto kg = key0;
    for (int k0 = 0; k0 < F; k0 += U) {
      // positions after frames k0..k0+U-1, then all their loads, then the merges
      bool in_c[U];
      uint32_t pos[U];
      uint32_t o[U], kk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) pos[u] = cell_of(k0 + u + 1, in_c[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool in_r = u == 0 ? in_prev : in_c[u - 1];
        const uint32_t r = u == 0 ? pos_prev : pos[u - 1];
        const bool ld = k0 + u < F && in_c[u] && in_r;
        const auto oa = og + r;
        const auto ka = kg + r;
        og += p.n;
        kg += p.n;
        o[u] = ld ? __ldcs(oa) : 0u;
        kk[u] = ld ? __ldcs(ka) : 0u;
      }
      uint32_t packed[U / 2] = {};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u;
        if (k >= F) break;
        const bool in_r = u == 0 ? in_prev : in_c[u - 1];
        if (in_c[u]) val = in_r ? merge_cell(val, decode_cell(o[u], kk[u], ep[k])) : 0u;  // shifted in: Unknown
        const unsigned oc = in_c[u] && val == 2u ? 1u : 0u, fr = in_c[u] && val == 1u ? 1u : 0u;
        packed[u >> 1] |= (oc | (fr << 8)) << (16 * (u & 1));
      }
      add_frame_counts<U>(packed, acc, k0, lane);
      // position after the group's last frame (F may end inside the group)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k0 + u < F) {
          in_prev = in_c[u];
          pos_prev = pos[u];
        }
      }
    }
    if (in_prev) dst[pos_prev] = static_cast<uint8_t>(val);
  }
  flush_frame_counts(acc, cnt, lane);
  __syncthreads();
  const unsigned long long t_end = global_ns();
  for (int k = threadIdx.x; k < F; k += blockDim.x) {
    Counters& c = p.counters[static_cast<long long>(s) * F + k];
    if (cnt[k]) atomicAdd(&c.occupied, static_cast<unsigned long long>(cnt[k]));
    if (cnt[kMaxFramesPerCall + k]) atomicAdd(&c.freed, static_cast<unsigned long long>(cnt[kMaxFramesPerCall + k]));
    atomicMax(&c.t_end, t_end);
  }
  if (p.k4_publish) chain_publish_when_last(p, s, F, vec_ok ? (nchain >> 2) : nchain);
}

template <bool kClear>
__global__ void __launch_bounds__(VXM_SEQ_THREADS) merge_sequence_kernel(KParams p, int F) {
  pdl_wait();  // K3's keys and counters
  constexpr int U = VXM_SEQ_U;  // frames whose loads are issued together
  __shared__ unsigned cnt[2 * kMaxFramesPerCall];           // occupied, then freed, per frame
  __shared__ int Pc[kMaxFramesPerCall + U][3];              // P_{k-1} at index k
  __shared__ uint32_t ep[kMaxFramesPerCall];
  const int s = blockIdx.y;  // stream
  const FrameParams* f0 = p.frames + static_cast<long long>(s) * F;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0) {
    const unsigned long long t = global_ns();
    for (int k = threadIdx.x; k < F; k += blockDim.x) p.counters[static_cast<long long>(s) * F + k].t_merge = t;
  }
  for (int k = threadIdx.x; k < 2 * kMaxFramesPerCall; k += blockDim.x) cnt[k] = 0u;
  __shared__ int vec_ok;
  if (threadIdx.x < 32) chain_prefix(f0, F, p.dx, Pc, ep, &vec_ok, lane);
  if (blockIdx.x == 0) {
    // fold the trace counters of every frame slot of this stream (one warp each)
    for (int k = threadIdx.x >> 5; k < F; k += blockDim.x >> 5) fold_trace_slots(p.counters[static_cast<long long>(s) * F + k]);
  }
  __syncthreads();
  const int dx = p.dx, dy = p.dy, dz = p.dz;
  const uint32_t dxy = static_cast<uint32_t>(dx) * static_cast<uint32_t>(dy);  // (cells < 2^32)
  const int bx = f0->box_lo[0], by = f0->box_lo[1], bz = f0->box_lo[2];
  const int ex = f0->box_ext[0], ey = f0->box_ext[1], ez = f0->box_ext[2];
  const long long nchain = static_cast<long long>(ex) * ey * ez;
  // blocks past the work (the grid is sized for the largest box) leave
  // before the counters: no idle t_end atomics on the frame slots
  if (blockIdx.x > 0 && static_cast<long long>(blockIdx.x) * blockDim.x >= (vec_ok ? (nchain >> 2) : nchain)) return;
  const uint32_t cur = f0->cur;
  const uint8_t* src = (cur ? p.loc1 : p.loc0) + static_cast<long long>(s) * p.n;
  uint8_t* dst = (cur ? p.loc0 : p.loc1) + static_cast<long long>(s) * p.n;
  const uint8_t* occ0 = p.occ + static_cast<long long>(s) * F * p.n;
  // clear format: every key a chain meets in the grid is read (also when the
  // cell shifts out of the grid afterwards) and reset to Unknown if touched,
  // so all F slots end all-Unknown
  uint32_t* key0 = p.key + static_cast<long long>(s) * F * p.n;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  uint32_t acc[4] = {0u, 0u, 0u, 0u};  // per-frame Occupied / Free counts, see add_frame_counts
  if (vec_ok) {
    // Every frame's x shift is a multiple of 4 (and dims_x too): a thread
    // folds 4 neighbouring chains at once, moving the 4 cells as one word
    // (occupancy u32, keys uint4) and merging / counting them with the
    // byte-SIMD helpers of K4.
    const int ex4 = ex >> 2;
    const long long ngroup = static_cast<long long>(ex4) * ey * ez;
    for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x; base < ngroup; base += stride) {
      const long long i = base + threadIdx.x;
      const bool active = i < ngroup;
      const int iz = static_cast<int>(i / (static_cast<long long>(ex4) * ey));
      const int rem = static_cast<int>(i - static_cast<long long>(iz) * ex4 * ey);
      const int iy = rem / ex4;
      const int gx = bx + 4 * (rem - iy * ex4), gy = by + iy, gz = bz + iz;
      auto group_of = [&](int k, bool& in) -> uint32_t {  // first cell of the group at c_{k-1}
        const int cx = gx - Pc[k][0], cy = gy - Pc[k][1], cz = gz - Pc[k][2];
        in = active && static_cast<unsigned>(cx) < static_cast<unsigned>(dx) &&
             static_cast<unsigned>(cy) < static_cast<unsigned>(dy) && static_cast<unsigned>(cz) < static_cast<unsigned>(dz);
        return static_cast<uint32_t>(cx) + static_cast<uint32_t>(cy) * static_cast<uint32_t>(dx) +
               static_cast<uint32_t>(cz) * dxy;
      };
      bool in_prev;
      uint32_t pos_prev = group_of(0, in_prev);
      uint32_t val = in_prev ? *reinterpret_cast<const uint32_t*>(src + pos_prev) : 0u;
      auto og = occ0;  // slabs of frame k0 (advanced one frame per load pair)
      auto kg = key0;
      for (int k0 = 0; k0 < F; k0 += U) {
        bool in_c[U];
        uint32_t pos[U];
        uint32_t o[U];
        uint4 kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) pos[u] = group_of(k0 + u + 1, in_c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool in_r = u == 0 ? in_prev : in_c[u - 1];
          const uint32_t r = u == 0 ? pos_prev : pos[u - 1];
          const bool ld = k0 + u < F && in_r && (kClear || in_c[u]);
          const auto oa = og + r;
          const auto ka = kg + r;
          og += p.n;
          kg += p.n;
          o[u] = ld && !kClear ? __ldcs(reinterpret_cast<const uint32_t*>(oa)) : 0u;
          kk[u] = ld ? __ldcs(reinterpret_cast<const uint4*>(ka)) : make_uint4(0u, 0u, 0u, 0u);
          if (kClear && ld && touched4(kk[u])) *reinterpret_cast<uint4*>(ka) = make_uint4(0u, 0u, 0u, 0u);
        }
        // per frame: Occupied / Free counts of this thread's 4 cells (each
        // <= 4, so a warp sum fits a byte); two frames share one reduction
        uint32_t packed[U / 2] = {};
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u;
          if (k >= F) break;
          const bool in_r = u == 0 ? in_prev : in_c[u - 1];
          if (in_c[u])  // shifted in: Unknown
            val = in_r ? merge4s(val, kClear ? states4_clear(kk[u]) : states4_epoch(o[u], kk[u], ep[k])) : 0u;
          const unsigned oc = in_c[u] ? count_occupied4(val) : 0u, fr = in_c[u] ? count_free4(val) : 0u;
          packed[u >> 1] |= (oc | (fr << 8)) << (16 * (u & 1));
        }
        add_frame_counts<U>(packed, acc, k0, lane);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (k0 + u < F) {
            in_prev = in_c[u];
            pos_prev = pos[u];
          }
        }
      }
      if (in_prev) *reinterpret_cast<uint32_t*>(dst + pos_prev) = val;
    }
  } else
  for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x; base < nchain; base += stride) {
    const long long i = base + threadIdx.x;
    const bool active = i < nchain;
    const int iz = static_cast<int>(i / (static_cast<long long>(ex) * ey));
    const int rem = static_cast<int>(i - static_cast<long long>(iz) * ex * ey);
    const int iy = rem / ex;
    const int gx = bx + rem - iy * ex, gy = by + iy, gz = bz + iz;
    auto cell_of = [&](int k, bool& in) -> uint32_t {  // c_{k-1} = g - P_{k-1}
      const int cx = gx - Pc[k][0], cy = gy - Pc[k][1], cz = gz - Pc[k][2];
      in = active && static_cast<unsigned>(cx) < static_cast<unsigned>(dx) &&
           static_cast<unsigned>(cy) < static_cast<unsigned>(dy) && static_cast<unsigned>(cz) < static_cast<unsigned>(dz);
      return static_cast<uint32_t>(cx) + static_cast<uint32_t>(cy) * static_cast<uint32_t>(dx) +
               static_cast<uint32_t>(cz) * dxy;
    };
    bool in_prev;
    uint32_t pos_prev = cell_of(0, in_prev);
    uint32_t val = in_prev ? src[pos_prev] : 0u;
    auto og = occ0;  // slabs of frame k0 (advanced one frame per load pair)
    auto kg = key0;
    for (int k0 = 0; k0 < F; k0 += U) {
      // positions after frames k0..k0+U-1, then all their loads, then the merges
      bool in_c[U];
      uint32_t pos[U];
      uint32_t o[U], kk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) pos[u] = cell_of(k0 + u + 1, in_c[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool in_r = u == 0 ? in_prev : in_c[u - 1];
        const uint32_t r = u == 0 ? pos_prev : pos[u - 1];
        const bool ld = k0 + u < F && in_r && (kClear || in_c[u]);
        const auto oa = og + r;
        const auto ka = kg + r;
        og += p.n;
        kg += p.n;
        o[u] = ld && !kClear ? __ldcs(oa) : 0u;
        kk[u] = ld ? __ldcs(ka) : 0u;
        if (kClear && kk[u]) *ka = 0u;
      }
      uint32_t packed[U / 2] = {};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u;
        if (k >= F) break;
        const bool in_r = u == 0 ? in_prev : in_c[u - 1];
        if (in_c[u])  // shifted in: Unknown
          val = in_r ? merge_cell(val, kClear ? decode_clear_key(kk[u]) : decode_cell(o[u], kk[u], ep[k])) : 0u;
        const unsigned oc = in_c[u] && val == 2u ? 1u : 0u, fr = in_c[u] && val == 1u ? 1u : 0u;
        packed[u >> 1] |= (oc | (fr << 8)) << (16 * (u & 1));
      }
      add_frame_counts<U>(packed, acc, k0, lane);
      // position after the group's last frame (F may end inside the group)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k0 + u < F) {
          in_prev = in_c[u];
          pos_prev = pos[u];
        }
      }
    }
    if (in_prev) dst[pos_prev] = static_cast<uint8_t>(val);
  }
  flush_frame_counts(acc, cnt, lane);
  __syncthreads();
  const unsigned long long t_end = global_ns();
  for (int k = threadIdx.x; k < F; k += blockDim.x) {
    Counters& c = p.counters[static_cast<long long>(s) * F + k];
    if (cnt[k]) atomicAdd(&c.occupied, static_cast<unsigned long long>(cnt[k]));
    if (cnt[kMaxFramesPerCall + k]) atomicAdd(&c.freed, static_cast<unsigned long long>(cnt[kMaxFramesPerCall + k]));
    atomicMax(&c.t_end, t_end);
  }
  if (p.k4_publish) chain_publish_when_last(p, s, F, vec_ok ? (nchain >> 2) : nchain);
}

}  // namespace vxm
