// 32x32->64 product forms on sm_100a: IMAD.WIDE.U32 vs IMAD + IMAD.HI.U32.
#include <cstdio>
typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u32 mulhi_asm(u32 a, u32 b) {
  u32 r; asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ u32 mullo_asm(u32 a, u32 b) {
  u32 r; asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ u64 mulwide_asm(u32 a, u32 b) {
  u64 r; asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b)); return r;
}

template <int KIND>
__global__ void probe(u32* out, u32 iters, u32 seed) {
  u32 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed * (i + 1) + threadIdx.x;
  const u32 b = seed | 1;
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (KIND == 0) { u64 w = mulwide_asm(a[i], b); a[i] = (u32)w ^ (u32)(w >> 32); }  // WIDE + LOP3
      if (KIND == 1) { a[i] = mullo_asm(a[i], b) ^ mulhi_asm(a[i], b); }                   // IMAD + IMAD.HI + LOP3
      if (KIND == 2) { a[i] = mulhi_asm(a[i], b) ^ a[i]; }                                 // IMAD.HI + LOP3
      if (KIND == 3) { a[i] = mullo_asm(a[i], b) ^ a[(i + 1) & 15]; }                      // IMAD + LOP3
    }
  }
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
float run(u32* out, u32 iters) {
  cudaEvent_t x, y; cudaEventCreate(&x); cudaEventCreate(&y);
  probe<KIND><<<148 * 8, 256>>>(out, 16, 7);
  cudaEventRecord(x);
  probe<KIND><<<148 * 8, 256>>>(out, iters, 7);
  cudaEventRecord(y); cudaEventSynchronize(y);
  float ms; cudaEventElapsedTime(&ms, x, y);
  return ms;
}

int main() {
  u32* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const u32 iters = 8192;
  const double warps = 148.0 * 8 * 256 / 32;
  const char* names[] = {"WIDE+LOP3", "IMAD+IMAD.HI+LOP3", "IMAD.HI+LOP3", "IMAD+LOP3"};
  float t[4] = {run<0>(out, iters), run<1>(out, iters), run<2>(out, iters), run<3>(out, iters)};
  for (int k = 0; k < 4; ++k) {
    const double ops = warps * iters * 16;
    printf("%-20s %.3f ms  %.3f ops/clk/SM\n", names[k], t[k], ops / (t[k] * 1e-3) / (clk * 1e3) / 148);
  }
  return 0;
}
