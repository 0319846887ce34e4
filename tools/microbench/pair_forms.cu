// Throughput probe for the pair-accumulation inner step (e = x - y, then
// e0^2, e0*e1, e1^2 summed exactly) in three arithmetic forms, register
// resident (no memory): pair-slots per clock per SM.
//   0: integer split-23 (10 IMAD.WIDE per pair-slot)
//   1: FP64 split-22 on integer-valued doubles (4 DADD + 10 DFMA)
//   2: mixed: squares on the FP64 pipe, the cross product on the integer pipe
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ void madw(u64& acc, u32 a, u32 b) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}
constexpr int P = 4;  // independent pair-slots per thread per iteration

template <int KIND>
__global__ void __launch_bounds__(256) probe(u64* out, u32 iters, u32 seed) {
  u64 xi0[P], xi1[P], xj0[P], xj1[P];
  double fh0[P], fl0[P], fh1[P], fl1[P], gh0[P], gl0[P], gh1[P], gl1[P];
#pragma unroll
  for (int t = 0; t < P; ++t) {
    xi0[t] = (seed * 977ull * (t + 1) + threadIdx.x) & ((1ull << 44) - 1);
    xi1[t] = xi0[t] ^ 0x5555555ull; xj0[t] = xi0[t] ^ 0x3333ull; xj1[t] = xi1[t] ^ 0x77777ull;
    fh0[t] = (double)(xi0[t] >> 22); fl0[t] = (double)(xi0[t] & 0x3FFFFF);
    fh1[t] = (double)(xi1[t] >> 22); fl1[t] = (double)(xi1[t] & 0x3FFFFF);
    gh0[t] = (double)(xj0[t] >> 22); gl0[t] = (double)(xj0[t] & 0x3FFFFF);
    gh1[t] = (double)(xj1[t] >> 22); gl1[t] = (double)(xj1[t] & 0x3FFFFF);
  }
  const u64 q = 17592182243329ull;
  u64 s[P][9];
  double d[P][10];
#pragma unroll
  for (int t = 0; t < P; ++t) {
#pragma unroll
    for (int k = 0; k < 9; ++k) s[t][k] = 0;
#pragma unroll
    for (int k = 0; k < 10; ++k) d[t][k] = 0;
  }
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < P; ++t) {
      if (KIND == 0) {
        const u64 e0 = xi0[t] - xj0[t] + q, e1 = xi1[t] - xj1[t] + q;
        const u32 l0 = (u32)e0 & 0x7FFFFF, h0 = (u32)(e0 >> 23);
        const u32 l1 = (u32)e1 & 0x7FFFFF, h1 = (u32)(e1 >> 23);
        madw(s[t][0], l0, l0); madw(s[t][1], l0, h0); madw(s[t][2], h0, h0);
        madw(s[t][3], l1, l1); madw(s[t][4], l1, h1); madw(s[t][5], h1, h1);
        madw(s[t][6], l0, l1); madw(s[t][7], l0, h1); madw(s[t][7], h0, l1); madw(s[t][8], h0, h1);
        xi0[t] += it; xj1[t] ^= it;  // keep the inputs live and varying
      }
      if (KIND == 1) {
        const double eh0 = fh0[t] - gh0[t], el0 = fl0[t] - gl0[t];
        const double eh1 = fh1[t] - gh1[t], el1 = fl1[t] - gl1[t];
        d[t][0] = fma(el0, el0, d[t][0]); d[t][1] = fma(eh0, el0, d[t][1]); d[t][2] = fma(eh0, eh0, d[t][2]);
        d[t][3] = fma(el1, el1, d[t][3]); d[t][4] = fma(eh1, el1, d[t][4]); d[t][5] = fma(eh1, eh1, d[t][5]);
        d[t][6] = fma(el0, el1, d[t][6]); d[t][7] = fma(el0, eh1, d[t][7]); d[t][8] = fma(eh0, el1, d[t][8]);
        d[t][9] = fma(eh0, eh1, d[t][9]);
        fh0[t] += 1.0; gl1[t] -= 1.0;
      }
      if (KIND == 2) {
        const double eh0 = fh0[t] - gh0[t], el0 = fl0[t] - gl0[t];
        const double eh1 = fh1[t] - gh1[t], el1 = fl1[t] - gl1[t];
        d[t][0] = fma(el0, el0, d[t][0]); d[t][1] = fma(eh0, el0, d[t][1]); d[t][2] = fma(eh0, eh0, d[t][2]);
        d[t][3] = fma(el1, el1, d[t][3]); d[t][4] = fma(eh1, el1, d[t][4]); d[t][5] = fma(eh1, eh1, d[t][5]);
        const u64 e0 = xi0[t] - xj0[t] + q, e1 = xi1[t] - xj1[t] + q;
        const u32 l0 = (u32)e0 & 0x7FFFFF, h0 = (u32)(e0 >> 23);
        const u32 l1 = (u32)e1 & 0x7FFFFF, h1 = (u32)(e1 >> 23);
        madw(s[t][6], l0, l1); madw(s[t][7], l0, h1); madw(s[t][7], h0, l1); madw(s[t][8], h0, h1);
        fh0[t] += 1.0; gl1[t] -= 1.0; xi0[t] += it; xj1[t] ^= it;
      }
    }
  }
  u64 r = 0;
#pragma unroll
  for (int t = 0; t < P; ++t) {
#pragma unroll
    for (int k = 0; k < 9; ++k) r ^= s[t][k];
#pragma unroll
    for (int k = 0; k < 10; ++k) r ^= (u64)d[t][k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int KIND>
float run(u64* out, u32 iters, int blocks) {
  cudaEvent_t x, y; cudaEventCreate(&x); cudaEventCreate(&y);
  probe<KIND><<<blocks, 256>>>(out, 16, 7);
  cudaEventRecord(x);
  probe<KIND><<<blocks, 256>>>(out, iters, 7);
  cudaEventRecord(y); cudaEventSynchronize(y);
  float ms; cudaEventElapsedTime(&ms, x, y);
  return ms;
}

int main() {
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"int split-23", "fp64 split-22", "mixed fp64 sq + int cross"};
  for (int occ : {2, 4, 8}) {
    const int blocks = 148 * occ;
    u64* out; cudaMalloc(&out, (size_t)blocks * 256 * 8);
    const u32 iters = 2048;
    float t[3] = {run<0>(out, iters, blocks), run<1>(out, iters, blocks), run<2>(out, iters, blocks)};
    for (int k = 0; k < 3; ++k) {
      const double ps = (double)blocks * 256 * iters * P;
      printf("occ %d x256  %-28s %.3f ms  %.2f pair-slots/clk/SM\n", occ, names[k], t[k],
             ps / (t[k] * 1e-3) / (clk * 1e3) / 148);
    }
    cudaFree(out);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
