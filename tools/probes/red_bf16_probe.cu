// Probe of the packed-bf16 max reduction (red.global.max.noftz.v2.bf16):
// for every ordered pair of 16-bit patterns from a sample (negative normals,
// negative/positive subnormals, zeros, positive normals, +-inf), initialise
// the low half of a word with `a`, reduce `b` into it (high half -inf), and
// compare the result with the IEEE maximum. Prints the mismatch count per
// class of (a, b).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

__global__ void red_kernel(uint32_t* w, const uint16_t* vals, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * n) return;
  uint16_t b = vals[i % n];
  uint32_t word = 0xFF800000u | b;
  asm volatile("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\t"
               "red.relaxed.gpu.global.max.noftz.v2.bf16 [%0], {lo, hi};\n\t}" ::"l"(w + i), "r"(word) : "memory");
}

static float bf(uint16_t p) { uint32_t u = uint32_t(p) << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
  std::vector<uint16_t> v;
  const uint16_t sample[] = {0xFF80, 0xFF7F, 0xFF7E, 0xFF7C, 0xFF00, 0xF000, 0xC000, 0x8081, 0x807F, 0x8003, 0x8002, 0x8001,
                             0x0000, 0x0001, 0x0002, 0x0003, 0x007F, 0x0080, 0x0081, 0x1000, 0x3F80, 0x7F7E, 0x7F7F, 0x7F80};
  for (uint16_t s : sample) v.push_back(s);
  const int n = v.size();
  uint32_t* dw; uint16_t* dv;
  cudaMalloc(&dw, 4 * n * n); cudaMalloc(&dv, 2 * n);
  cudaMemcpy(dv, v.data(), 2 * n, cudaMemcpyHostToDevice);
  std::vector<uint32_t> init(n * n);
  for (int i = 0; i < n * n; ++i) init[i] = 0xFF800000u | v[i / n];
  cudaMemcpy(dw, init.data(), 4 * n * n, cudaMemcpyHostToDevice);
  red_kernel<<<(n * n + 127) / 128, 128>>>(dw, dv, n);
  std::vector<uint32_t> out(n * n);
  cudaMemcpy(out.data(), dw, 4 * n * n, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n * n; ++i) {
    uint16_t a = v[i / n], b = v[i % n];
    float fa = bf(a), fb = bf(b);
    uint16_t want = fa > fb ? a : (fb > fa ? b : (a == b ? a : 0xFFFF));  // +0/-0 tie: either
    uint16_t got = out[i] & 0xFFFF;
    uint16_t hi = out[i] >> 16;
    if ((want != 0xFFFF && got != want) || hi != 0xFF80) {
      if (bad < 40) printf("a=%04x b=%04x got=%04x want=%04x hi=%04x\n", a, b, got, want, hi);
      ++bad;
    }
  }
  printf("pairs %d mismatches %d\n", n * n, bad);
  return 0;
}
