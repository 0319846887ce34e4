// FP64 vs integer pipe probe on sm_100a: is the FP64 pipe a second modular
// multiplier? Independent chains, register-resident; prints butterflies (or
// ops) per clock per SM.
//   KIND 0: DFMA chains                       (raw FP64 rate)
//   KIND 1: FP64 CT butterfly (exact integer-valued doubles, q < 2^45)
//   KIND 2: integer CT butterfly (truncated Shoup, the ntt.cuh ct_bfly)
//   KIND 3: half the chains KIND 1, half KIND 2 (do the pipes overlap?)
#include <cstdint>
#include <cstdio>
typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u64 mul_shoup_lazy4(u64 a, u64 w, u64 ws, u64 q) {
  const u32 a0 = (u32)a, a1 = (u32)(a >> 32);
  const u32 s0 = (u32)ws, s1 = (u32)(ws >> 32);
  const u64 t1 = (u64)a1 * s0, t2 = (u64)a0 * s1;
  const u64 hi = (u64)a1 * s1 + (t1 >> 32) + (t2 >> 32);
  return a * w - hi * q;
}

// t = y * w mod q (signed lazy, |t| < 2q) for integer-valued doubles.
__device__ __forceinline__ double mulmod_f64(double y, double w, double wq, double q) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  const double ph = __dmul_rn(y, w);
  const double pl = __fma_rn(y, w, -ph);
  const double qt = __dadd_rn(__fma_rn(y, wq, M), -M);
  const double r = __fma_rn(-qt, q, ph);
  return __dadd_rn(r, pl);
}

template <int KIND>
__global__ void probe(u64* out, u32 iters, u32 seed) {
  constexpr int C = 16;
  double xf[C];
  u64 xi[C];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    xi[i] = (u64)(seed * (i + 1) + threadIdx.x) * 977ull;
    xf[i] = (double)(xi[i] & 0xFFFFFFFFFFull);
  }
  const double q = 17592182243329.0, w = 1234567891011.0, wq = w / q;
  const u64 qi = 17592182243329ull, wi = 1234567891011ull;
  const u64 ws = (u64)(((unsigned __int128)wi << 64) / qi);
  for (u32 it = 0; it < iters; ++it) {
    if (KIND == 0) {
#pragma unroll
      for (int i = 0; i < C; ++i) xf[i] = __fma_rn(xf[i], wq, xf[(i + 1) & (C - 1)]);
    }
    if (KIND == 1 || KIND == 3) {
      constexpr int E = KIND == 1 ? C : C / 2;
#pragma unroll
      for (int i = 0; i < E / 2; ++i) {
        const double t = mulmod_f64(xf[2 * i + 1], w, wq, q);
        const double a = xf[2 * i];
        xf[2 * i] = a + t;
        xf[2 * i + 1] = a - t;
      }
    }
    if (KIND == 2 || KIND == 3) {
      constexpr int B = KIND == 2 ? 0 : C / 2;
#pragma unroll
      for (int i = B / 2; i < C / 2; ++i) {
        const u64 t = mul_shoup_lazy4(xi[2 * i + 1], wi, ws, qi);
        const u64 a = xi[2 * i];
        xi[2 * i] = a + t;
        xi[2 * i + 1] = a + (4 * qi - t);
      }
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += xi[i] + (u64)__double_as_longlong(xf[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
float run(u64* out, u32 iters, int blocks_per_sm, int threads) {
  cudaEvent_t x, y;
  cudaEventCreate(&x);
  cudaEventCreate(&y);
  probe<KIND><<<148 * blocks_per_sm, threads>>>(out, 16, 7);
  cudaEventRecord(x);
  probe<KIND><<<148 * blocks_per_sm, threads>>>(out, iters, 7);
  cudaEventRecord(y);
  cudaEventSynchronize(y);
  float ms;
  cudaEventElapsedTime(&ms, x, y);
  return ms;
}

int main() {
  u64* out;
  cudaMalloc(&out, 148 * 16 * 256 * 8);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const u32 iters = 2048;
  for (int occ : {4, 8}) {
    const double threads = 148.0 * occ * 256;
    const double per = threads * iters / 148.0 / (clk * 1e3);  // per-SM thread-iterations per ms-clock
    float t0 = run<0>(out, iters, occ, 256), t1 = run<1>(out, iters, occ, 256);
    float t2 = run<2>(out, iters, occ, 256), t3 = run<3>(out, iters, occ, 256);
    printf("occupancy %d x 256 threads/SM (clock %d kHz)\n", occ, clk);
    printf("  DFMA             %.3f ms  %.1f thread-ops/clk/SM\n", t0, 16 * per / t0);
    printf("  fp64 butterfly   %.3f ms  %.2f bfly/clk/SM\n", t1, 8 * per / t1);
    printf("  int butterfly    %.3f ms  %.2f bfly/clk/SM\n", t2, 8 * per / t2);
    printf("  mixed 4+4        %.3f ms  %.2f bfly/clk/SM\n", t3, 8 * per / t3);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
