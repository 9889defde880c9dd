// Device-side data layout and arithmetic shared by every voxmap kernel.
//
// Bit-exactness contract: the reference computes in
// fp64 with IEEE add/mul/div/sqrt, no FMA contraction (built with
// -ffp-contract=off, proj/src/CMakeLists.txt:33-35) and a fixed operation
// order. Every fp64 operation below is spelled with a _rn intrinsic so the
// compiler can neither contract nor reorder it; the library is also built
// with -fmad=false as a second guard.
#pragma once

#include <cstdint>

namespace vxm {

// ---------------------------------------------------------------------------
// Measurement-grid words.
//
// The reference measurement grid is one byte per cell, reset to Unknown every
// frame (proj/src/pipeline.cpp:83), written Occupied by populate and Free /
// UnknownTraced by the rays, with the highest-index ray winning a conflict in
// Sequential mode (raytracer.cpp:98-104). On the GPU each cell
// is one 32-bit word whose top bits carry a per-stream frame epoch:
//
//   word = epoch << 18 | low18
//   low18 == 0x3FFFF                  Occupied
//   low18 == (ray + 1) << 1 | traced  written by bundle ray `ray`
//   low18 == 0 / 1                    Free / UnknownTraced carried in from a
//                                     host grid (lowest priority)
//   epoch != current epoch            Unknown (no per-frame reset needed)
//
// Populate stores the Occupied word with plain stores (idempotent, no
// atomics). Rays resolve conflicts with a fire-and-forget atomicMax: a higher
// ray index always wins, exactly the Sequential last-writer rule, and the
// Occupied word is the maximum of its epoch so rays can never overwrite it.
// ---------------------------------------------------------------------------
constexpr uint32_t kEpochShift = 18;
constexpr uint32_t kLowMask = (1u << kEpochShift) - 1u;  // 0x3FFFF
constexpr uint32_t kMaxEpoch = (1u << (32 - kEpochShift)) - 1u;
constexpr uint32_t kMaxRays = (kLowMask >> 1) - 1u;  // (ray+1)<<1|1 < 0x3FFFF

__host__ __device__ constexpr uint32_t occupied_word(uint32_t tag) { return tag | kLowMask; }

// Word -> reference byte state (0 Unknown, 1 Free, 2 Occupied, 3 UnknownTraced).
__device__ __forceinline__ uint32_t decode_word(uint32_t w, uint32_t tag) {
  if ((w & ~kLowMask) != tag) return 0u;
  const uint32_t low = w & kLowMask;
  if (low == kLowMask) return 2u;
  return (low & 1u) ? 3u : 1u;
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
};

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
  int32_t off[3];     // shift applied after the merge (0,0,0 = none)
  uint32_t tag;       // epoch << 18
  uint32_t cur;       // which local buffer holds the current grid
  uint32_t pad_;
};

// Constant (per-context) launch parameters, passed by value.
struct KParams {
  // grid
  int dx, dy, dz;
  long long n;        // cells per stream
  double vs;
  // camera (host-computed with glibc tan, never recomputed on device)
  int W, H;
  double fx, fy, cx, cy, max_depth;
  // populate
  int vox_inf;
  // bundle
  int vd, vw, vh;
  int tiles_x, tiles_y;  // 8x4 ray tiles per warp
  // buffers (stream s at offset s*n)
  uint32_t* msw;       // measurement words (occupied / ray keys)
  uint32_t* ctr;       // centre words when vox_inf > 0
  uint8_t* loc0;
  uint8_t* loc1;
  Counters* counters;
  const FrameParams* frames;
};

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
__device__ __forceinline__ int voxel_coord(double acc, double vs) {
  double f = floor(ddiv(acc, vs));
  f = (f < -1e9) ? -1e9 : f;
  f = (1e9 < f) ? 1e9 : f;
  if (f != f) return INT32_MIN;
  return static_cast<int>(f);
}

// p_v[a] = ((t[a] + R[3a]x) + R[3a+1]y) + R[3a+2]z   (kernels_scalar.cpp:27-30)
__device__ __forceinline__ void transform_voxelize(const double* R, const double* t, double x,
                                                   double y, double z, double vs, int* c) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double acc = t[a];
    acc = dadd(acc, dmul(R[3 * a + 0], x));
    acc = dadd(acc, dmul(R[3 * a + 1], y));
    acc = dadd(acc, dmul(R[3 * a + 2], z));
    c[a] = voxel_coord(acc, vs);
  }
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned v) {
  return __reduce_add_sync(0xffffffffu, v);
}

// Block-wide sums of up to 4 counters; thread 0 adds them to global memory.
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

}  // namespace vxm
