// Integer pipe throughput probe on sm_100a: independent chains of one
// instruction type; prints warp-instructions per clock per SM.
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
typedef unsigned int u32;

template <int KIND>
__global__ void probe(u64* out, u32 iters, u32 seed) {
  u32 a[16]; u64 w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = seed * (i + 1) + threadIdx.x; w[i] = a[i] * 3ull; }
  const u32 b = seed | 1;
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (KIND == 0) w[i] = (u64)(u32)(w[i] >> 17) * b + w[(i + 1) & 15];  // IMAD.WIDE.U32 (acc) + SHF
      if (KIND == 5) a[i] = __umulhi(a[i], b) + a[(i + 1) & 15];  // IMAD.HI
      if (KIND == 1) a[i] = a[i] * b + a[(i + 1) & 15];           // IMAD
      if (KIND == 2) a[i] = a[i] + b + a[(i + 3) & 15];           // IADD3
      if (KIND == 3) w[i] = w[i] + (w[(i + 1) & 15] ^ b);         // 64-bit add (IADD3 + IADD3.X) + LOP3
      if (KIND == 4) w[i] = __umul64hi(w[i], w[(i + 5) & 15]) + w[i]; // 64x64 hi
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += w[i] + a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
float run(u64* out, u32 iters) {
  cudaEvent_t x, y; cudaEventCreate(&x); cudaEventCreate(&y);
  probe<KIND><<<148 * 8, 256>>>(out, 16, 7);
  cudaEventRecord(x);
  probe<KIND><<<148 * 8, 256>>>(out, iters, 7);
  cudaEventRecord(y); cudaEventSynchronize(y);
  float ms; cudaEventElapsedTime(&ms, x, y);
  return ms;
}

int main() {
  u64* out; cudaMalloc(&out, 148 * 8 * 256 * 8);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const u32 iters = 4096;
  const double warps = 148.0 * 8 * 256 / 32;
  const char* names[] = {"IMAD.WIDE+SHF", "IMAD", "IADD3", "u64 add+xor", "umul64hi", "IMAD.HI+IADD"};
  float t[6] = {run<0>(out, iters), run<1>(out, iters), run<2>(out, iters), run<3>(out, iters), run<4>(out, iters), run<5>(out, iters)};
  for (int k = 0; k < 6; ++k) {
    const double ops = warps * iters * 16;  // warp-level source ops
    const double per_clk_sm = ops / (t[k] * 1e-3) / (clk * 1e3) / 148;
    printf("%-20s %.3f ms  %.2f source-ops/clk/SM (warp)\n", names[k], t[k], per_clk_sm);
  }
  return 0;
}
