// Device-side data layout and arithmetic shared by every voxmap kernel.
//
// Bit-exactness contract: the reference computes in
// fp64 with IEEE add/mul/div/sqrt, no FMA contraction (built with
// -ffp-contract=off, proj/src/CMakeLists.txt:33-35) and a fixed operation
// order. Every fp64 operation below is spelled with a _rn intrinsic so the
// compiler can neither contract nor reorder it; the library is also built
// with -fmad=false as a second guard.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace vxm {

// ---------------------------------------------------------------------------
// Measurement grid on the GPU.
//
// The reference measurement grid is one byte per cell, reset to Unknown every
// frame (proj/src/pipeline.cpp:83), written Occupied by populate and Free /
// UnknownTraced by the rays, with the highest-index ray winning a conflict in
// Sequential mode (raytracer.cpp:98-104). The GPU keeps two
// arrays per measurement slot, never reset as a whole:
//
//   occ[c]  (uint8)  == e   Occupied this frame (e = the slot's 8-bit epoch,
//                            1..255; a slot's arrays are cleared once per 255
//                            frames). Read-only during the trace.
//   key[c]  (uint32)         the cell's ray write as an ordered key; a ray
//                            writes key(ray) | traced with a fire-and-forget
//                            RED.max, so the highest ray index wins: exactly
//                            the Sequential last-writer rule.
//
// Two key formats (KeyFmt):
//   kEpochKeys (bundles of up to 131,070 rays, every BASELINE config):
//     key = e << 18 | (ray + 1) << 1 | traced; keys of another epoch read as
//     Unknown, so nothing is reset between frames; Free / UnknownTraced
//     carried in from a host grid are e << 18 | 0 / 1 (below every ray).
//     The merge reads occ (Occupied wins) and the keys.
//   kClearKeys (larger bundles, up to 2^31 - 3 rays; the reference has no
//     cap): Unknown 0 < carried Free 2 / UnknownTraced 3 < ray r: 2(r + 2) |
//     traced < Occupied 0xFFFFFFFF (stored by populate / dilation). The merge
//     decodes the keys alone and writes Unknown back over every key it saw
//     touched and over the cells the shift drops, so the slot is all-Unknown
//     when the next frame starts.
// Measured (B200, 64 cfg2 streams): the clearing writes cost the merge more
// than skipping the occupancy reads saves (K4 60 vs 50 us), and 16-bit keys
// ordered as bf16 patterns (packed-bf16 RED.max; K4 52 us) added ~10 us of
// resolve instructions to the ray cast, so the epoch format stays the
// default and the clear format only lifts the bundle limit.
// ---------------------------------------------------------------------------
enum KeyFmt : int { kEpochKeys = 0, kClearKeys = 1 };

constexpr uint32_t kKeyShift = 18;                     // epoch keys
constexpr uint32_t kLowMask = (1u << kKeyShift) - 1u;  // 0x3FFFF
constexpr uint32_t kMaxEpoch = 255u;                   // fits the occ byte
constexpr long long kMaxEpochRays = (kLowMask >> 1) - 1u;  // (ray+1)<<1|1 <= 0x3FFFD: 131,070 rays
constexpr long long kMaxClearRays = 0x7FFFFFFDLL;          // 2(ray+2)|1 < 0xFFFFFFFF
constexpr uint32_t kClearOccupied = 0xFFFFFFFFu;
constexpr int kMaxVoxInf = 16;  // the tile dilation (K2); larger radii take the generic passes

__host__ __device__ constexpr uint32_t key_tag(uint32_t epoch) { return epoch << kKeyShift; }

// Free key of ray r (| 1: UnknownTraced); r = -1: carried in from a host grid
__host__ __device__ __forceinline__ uint32_t ray_key(int fmt, uint32_t epoch, long long r) {
  return fmt == kEpochKeys ? key_tag(epoch) | static_cast<uint32_t>((r + 1) << 1) : static_cast<uint32_t>(2 * (r + 2));
}

// (occ, key) -> reference byte state (0 Unknown, 1 Free, 2 Occupied, 3 UnknownTraced).
__host__ __device__ __forceinline__ uint32_t decode_cell(uint32_t occ, uint32_t key, uint32_t epoch) {
  if (occ == epoch) return 2u;
  if ((key >> kKeyShift) != epoch) return 0u;
  return (key & 1u) ? 3u : 1u;
}
__host__ __device__ __forceinline__ uint32_t decode_clear_key(uint32_t k) {
  return k == 0u ? 0u : (k == kClearOccupied ? 2u : 1u + 2u * (k & 1u));
}

// merge_scalar (proj/src/kernels/kernels_scalar.cpp:10-16): measurement 0
// keeps the local cell, 3 writes Unknown, anything else is copied through.
__host__ __device__ __forceinline__ uint32_t merge_cell(uint32_t local, uint32_t m) {
  return m == 0u ? local : (m == 3u ? 0u : m);
}

// Per-stream counters, accumulated with one atomic per block.
struct Counters {
  unsigned long long points_total;
  unsigned long long points_outside;
  unsigned long long rays_traced;
  unsigned long long voxels_freed;
  unsigned long long voxels_traced;
  unsigned long long voxels_skipped;
  unsigned long long occupied;
  unsigned long long freed;
  // %globaltimer stamps (ns) of the stage starts for this slot: populate
  // (K1 block 0), trace and merge (block 0, once the previous stage has
  // completed), and the merge's end (max over its blocks); the host turns
  // them into vxm_stats::*_us without event nodes in the frame graph
  unsigned long long t_pop, t_trace, t_merge, t_end;
  unsigned long long trace_slots[32][4];  // K3 partials, folded by K4 (device only)
  unsigned long long merge_done;          // K4 blocks finished (the last one publishes)
  // K1: the smallest camera distance lower bound over this frame's points
  // (float bits, atomicMin; +inf after each publish, 0 = unknown): the ray
  // cast needs no occupancy reads for steps closer than that (minus the
  // dilation radius)
  unsigned int min_dist_bits;
  // K1 (dense depth): warps of this slot's K1 that found their first tile
  // face-heavy (low half, this frame; moved to the high half at the publish),
  // read by the next K1 of the slot to start such warps one pixel at a time.
  // A hint only: every mode gives the same result.
  unsigned int pop_faces;
};

// Per-warp min of a non-negative float, folded into *dst (as ordered bits).
__device__ __forceinline__ void warp_min_dist(float v, unsigned int* dst) {
  const unsigned b = __reduce_min_sync(0xffffffffu, __float_as_uint(v));
  if ((threadIdx.x & 31) == 0 && b != 0x7F800000u) atomicMin(dst, b);
}
// The part of Counters the host reads back: K5 copies it into host-mapped
// memory and clears the slot's Counters for the next frame.
struct CountersHead {
  unsigned long long points_total, points_outside, rays_traced, voxels_freed, voxels_traced, voxels_skipped,
      occupied, freed, t_pop, t_trace, t_merge, t_end;
};
static_assert(sizeof(CountersHead) == offsetof(Counters, trace_slots), "CountersHead mirrors Counters");
constexpr size_t kCountersHostBytes = sizeof(CountersHead);

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-stream, per-frame parameters: uploaded each frame as one small H2D
// copy so that the captured CUDA graph never changes.
struct FrameParams {
  double rot[9];      // R_vc = R_wc, row-major
  double trans[3];    // t_vc = t_wc - origin (camera centre in grid frame)
  const float* depth; // this stream's depth frame in device memory
  const double* xs;   // or a camera-frame cloud (cloud path)
  const double* ys;
  const double* zs;
  long long n_points;
  // this stream's occupancy bytes and keys (base + slot*n); read from memory
  // so the tracer keeps them in registers instead of rebuilding each address
  const uint8_t* occ_s;
  uint32_t* key_s;
  int32_t off[3];     // shift applied after the merge (0,0,0 = none)
  uint32_t epoch;     // 1..255
  uint32_t cur;       // which local buffer holds the current grid
  // multi-frame calls (frames_per_call > 1), first slot of a stream only:
  // the box of chain coordinates g = cell + P_k (P_k = sum of the shifts of
  // frames 0..k) that some frame's grid covers (merge_sequence_kernel)
  int32_t box_lo[3];
  int32_t box_ext[3];
  // per-frame constants of every ray's walk set-up (walk_ray,
  // raytracer.hpp:80-98), computed once on the host with the same IEEE
  // operations: the camera's cell floor(t_vc / vs) and the tmax numerators
  // (cur + 1) vs - t_vc (positive directions) and cur vs - t_vc (negative)
  int32_t cam_cell[3];
  uint32_t pad_;
  double tnum_pos[3];
  double tnum_neg[3];
};

// The largest float not above m (exact test of a float depth against a
// double range: (double)d > m  <=>  d > max_float_at_most(m)).
inline float max_float_at_most(double m) {
  float f = static_cast<float>(m);
  if (static_cast<double>(f) > m) f = std::nextafter(f, -INFINITY);
  return f;
}

// Fills FrameParams::cam_cell / tnum_* from f.trans and the walk's voxel
// size (host side; the kernels read them instead of dividing per ray).
inline void set_ray_consts(FrameParams& f, double vs) {
  for (int a = 0; a < 3; ++a) {
    const volatile double q = f.trans[a] / vs;  // (volatile: no contraction or reordering)
    f.cam_cell[a] = static_cast<int>(std::floor(q));
    const volatile double hp = static_cast<double>(f.cam_cell[a] + 1) * vs;
    const volatile double hn = static_cast<double>(f.cam_cell[a]) * vs;
    f.tnum_pos[a] = hp - f.trans[a];
    f.tnum_neg[a] = hn - f.trans[a];
  }
}

// Constant (per-context) launch parameters, passed by value.
struct KParams {
  // grid
  int dx, dy, dz;
  long long n;        // cells per stream
  double vs;
  double ray_vs;      // vox_size given to generate_rays (== vs on the pipeline path)
  double inv_vs;      // RN(1 / vs), fast-path divisor (see voxel_coord)
  // camera
  int W, H;
  double max_depth;
  float max_depth_f;  // the largest float <= max_depth: for a float depth d,
                      // (double)d > max_depth exactly when d > max_depth_f
  const double* qx;   // ((u + 0.5) - cx) / fx per column (host glibc tan)
  const double* qy;   // ((v + 0.5) - cy) / fy per row
  // populate
  int vox_inf;
  // bundle
  int vd, vw, vh;
  int tiles_x, tiles_y;  // 8x4 ray tiles per warp
  // buffers (stream s at offset s*n)
  uint8_t* occ;
  uint8_t* ctr;        // centre bytes when vox_inf > 0
  uint8_t* rowflag;    // [dy*dz] per slot: == epoch when the x-row holds a centre (vox_inf > 0)
  uint32_t* dbits;     // x-dilated centre bit rows [dy*dz][row words] (vox_inf > 0)
  uint8_t* dtmp;       // generic dilation (large radii / rows): 2 * n bytes per slot
  uint32_t* key;
  int key_fmt;         // KeyFmt
  int k4_publish;      // K4's last block per slot publishes the counters (no K5)
  uint8_t* loc0;
  uint8_t* loc1;
  Counters* counters;
  CountersHead* counters_out;  // host-mapped read-back (K5)
  const FrameParams* frames;
};

// 0xff in every byte of x that is zero, 0x00 elsewhere (exact, no carries
// across bytes: each byte's low 7 bits + 0x7f stays within the byte).
// 0x80 in every byte of x that is zero, 0 elsewhere
__device__ __forceinline__ uint32_t zero_bytes_msb(uint32_t x) {
  return ((((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u) ^ 0x80808080u;
}
__device__ __forceinline__ uint32_t zero_bytes(uint32_t x) {
  const uint32_t nonzero = (((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
  return ((nonzero ^ 0x80808080u) >> 7) * 0xffu;
}

// Occupied key at cell idx (populate / dilation): the clear format decodes
// occupancy from the keys; the epoch format from occ (storing its Occupied
// key as well, so that the trace could read occupancy from the key word,
// made the ray cast 10% slower: 4x the L1 footprint of the byte loads)
__device__ __forceinline__ void store_occupied_key(uint32_t* key, uint32_t idx, int fmt) {
  if (fmt == kClearKeys) key[idx] = kClearOccupied;
}

// Measurement states (bytes 0..3) of 4 consecutive cells from their
// occupancy bytes o4 and keys (epoch format) ...
__device__ __forceinline__ uint32_t states4_epoch(uint32_t o4, uint4 k4, uint32_t epoch) {
  const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
  uint32_t m4 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t v = (kk[i] >> kKeyShift) == epoch ? (1u | ((kk[i] & 1u) << 1)) : 0u;  // 1 or 3
    m4 |= v << (8 * i);
  }
  const uint32_t occm = zero_bytes(o4 ^ (epoch * 0x01010101u));  // 0xff where Occupied
  return (m4 & ~occm) | (0x02020202u & occm);
}
// ... or from the keys alone (clear format).
__device__ __forceinline__ uint32_t states4_clear(uint4 k) {
  return decode_clear_key(k.x) | (decode_clear_key(k.y) << 8) | (decode_clear_key(k.z) << 16) |
         (decode_clear_key(k.w) << 24);
}
__device__ __forceinline__ bool touched4(uint4 k) { return (k.x | k.y | k.z | k.w) != 0u; }

// merge of 4 packed cells: local l4 and measurement states m4 (bytes 0..3,
// so "== 0" and "== 3" are two-bit tests): merge_cell per byte.
__device__ __forceinline__ uint32_t merge4s(uint32_t l4, uint32_t m4) {
  const uint32_t keep = (((m4 | (m4 >> 1)) & 0x01010101u) ^ 0x01010101u) * 0xffu;  // m == 0
  const uint32_t clear = (m4 & (m4 >> 1) & 0x01010101u) * 0xffu;                   // m == 3
  return (l4 & keep) | (m4 & ~(keep | clear));
}

// ---------------------------------------------------------------------------
// fp64 helpers, each a single IEEE-rounded operation.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// floor(acc / vs), clamped to +-1e9 and truncated to int32, exactly as
// transform_voxelize_scalar (proj/src/kernels/kernels_scalar.cpp:31-34):
// f = std::min(std::max(f, -1e9), 1e9) keeps NaN, and x86's cvttsd2si turns
// NaN into INT32_MIN, which the bounds test then rejects.
__device__ __noinline__ int voxel_coord_exact(double acc, double vs) {
  double f = floor(ddiv(acc, vs));
  f = (f < -1e9) ? -1e9 : f;
  f = (1e9 < f) ? 1e9 : f;
  if (f != f) return INT32_MIN;
  return static_cast<int>(f);
}

// Same value without the IEEE division whenever that is provable:
// q = RN(acc * RN(1/vs)) is within 2^-51 |q| of RN(acc/vs). For |q| < 2^29
// (inside the +-1e9 clamp) that is below 2^-22, so when q's fractional part
// lies in (2^-16, 1 - 2^-16) both quotients share their floor. floor(q)
// comes from one round-down add of 1.5*2^52 (exact: the sum is an integer in
// [2^52, 2^53)), its int32 value is the sum's low word, and the range and
// fraction tests read the high words, so the fast path costs four fp64
// operations and a few integer compares. Otherwise (near an integer, zero,
// large, NaN) the exact division runs.
// Near an integer (where the fast path declines: points on voxel faces, e.g.
// axis-aligned walls, land within a few ulps of one) the floor is still
// decided without the division: with k = rint(q), |Q - k| < 2^-15 for the
// exact quotient Q = acc / vs, so floor(RN(Q)) is k or k - 1, and RN(Q) >= k
// iff Q >= k - d/2, d = k - nextafter(k, -inf) (a tie rounds to k: an integer
// below 2^29 has an even significand), i.e. iff acc - k vs >= -(d/2) vs.
// r = fma(-k, vs, acc) and hv = RN((d/2) vs) (d/2 is exact) are each within
// 2^-53 of their exact values, so the sign of e = r + hv is that of the exact
// expression whenever |e| > 2^-49 (|r| + hv). Otherwise (a quotient at a
// rounding midpoint), k == 0 (d/2 underflows) or NaN: ok = false.
__device__ __forceinline__ int voxel_coord_near(double acc, double q, double vs, bool& ok) {
  const double k = rint(q);
  const long long kb = __double_as_longlong(k);
  const double pk = __longlong_as_double(k > 0.0 ? kb - 1 : kb + 1);  // nextafter(k, -inf), k != 0
  const double hv = dmul(dmul(dsub(k, pk), 0.5), vs);
  const double r = __fma_rn(-k, vs, acc);
  const double e = dadd(r, hv);
  ok = k != 0.0 && fabs(e) > dmul(dadd(fabs(r), hv), 0x1p-49);
  return static_cast<int>(k) - (e < 0.0 ? 1 : 0);
}

// The fast path alone (then the near-integer test): ok = false when the exact
// division must decide.
__device__ __forceinline__ int voxel_coord_fast(double acc, double vs, double inv_vs, bool& ok) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double q = dmul(acc, inv_vs);
  const double t = __dadd_rd(q, kMagic);
  const double frac = dsub(q, dsub(t, kMagic));
  const uint32_t qhi = static_cast<uint32_t>(__double2hiint(q)) & 0x7fffffffu;
  const uint32_t fhi = static_cast<uint32_t>(__double2hiint(frac));
  ok = qhi < 0x41C00000u && fhi > 0x3EF00000u && fhi < 0x3FEFFFE0u;
  return __double2loint(t);
}

// where the fast path declined: the near-integer test, else the division
__device__ __forceinline__ int voxel_coord_slow(double acc, double vs, double inv_vs) {
  const double q = dmul(acc, inv_vs);
  const uint32_t qhi = static_cast<uint32_t>(__double2hiint(q)) & 0x7fffffffu;
  if (qhi < 0x41C00000u) {  // (|q| >= 2^29 or NaN: the clamp and NaN rules of the exact path)
    bool ok;
    const int c = voxel_coord_near(acc, q, vs, ok);
    if (ok) return c;
  }
  return voxel_coord_exact(acc, vs);
}

__device__ __forceinline__ int voxel_coord(double acc, double vs, double inv_vs) {
  bool ok;
  const int c = voxel_coord_fast(acc, vs, inv_vs, ok);
  return ok ? c : voxel_coord_slow(acc, vs, inv_vs);
}

// p_v[a] = ((t[a] + R[3a]x) + R[3a+1]y) + R[3a+2]z   (kernels_scalar.cpp:27-30)
// (slow: set when a coordinate needed more than the fast floor)
__device__ __forceinline__ void transform_voxelize(const double* R, const double* t, double x,
                                                   double y, double z, double vs,
                                                   double inv_vs, int* c, bool* slow = nullptr) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double acc = t[a];
    acc = dadd(acc, dmul(R[3 * a + 0], x));
    acc = dadd(acc, dmul(R[3 * a + 1], y));
    acc = dadd(acc, dmul(R[3 * a + 2], z));
    bool ok;
    int f = voxel_coord_fast(acc, vs, inv_vs, ok);
    if (!ok) {
      if (slow) *slow = true;
      f = voxel_coord_slow(acc, vs, inv_vs);
    }
    c[a] = f;
  }
}

// Warp-wide sums of NC counters; one atomic per counter per warp (no block
// barrier, so a warp with little work exits at once).
template <int NC>
__device__ __forceinline__ void warp_accumulate(unsigned (&v)[NC], unsigned long long* dst[NC]) {
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const unsigned s = __reduce_add_sync(0xffffffffu, v[i]);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(dst[i], static_cast<unsigned long long>(s));
  }
}

// Block-wide sums of NC counters; one atomic per counter per block.
template <int NC>
__device__ __forceinline__ void block_accumulate(unsigned (&v)[NC], unsigned long long* dst[NC]) {
  __shared__ unsigned long long partial[NC][32];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const unsigned s = __reduce_add_sync(0xffffffffu, v[i]);
    if (lane == 0) partial[i][warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      unsigned long long s = lane < nwarps ? partial[i][lane] : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0 && s) atomicAdd(dst[i], s);
    }
  }
}


// ---------------------------------------------------------------------------
// Bulk asynchronous copies (TMA engine, cp.async.bulk) into shared memory,
// completed on an mbarrier with a transaction byte count.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// makes the barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// the same with an L2 evict-first policy (data read once: the depth frames)
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 pol;\n\t"
               "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
               "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n\t}"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred p;\n\t"
               "WAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra WAIT_%=;\n\t}"
               ::"r"(smem_u32(bar)), "r"(phase)
               : "memory");
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while the previous kernel on its stream drains; it runs its independent
// prologue, then pdl_wait() blocks until that kernel has completed and its
// writes are visible (a no-op for an ordinary launch).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Kernel launch with programmatic dependent launch on or off (launch
// priorities for the memory-bound stages over the ray cast were measured too:
// no effect on the desynchronised batch, so every launch uses the default).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  return launch_ex(true, kernel, grid, block, smem, st, args...);
}

}  // namespace vxm
