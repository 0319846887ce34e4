// Client side of a round: pack_and_encrypt (distance.cpp:64-91)
// = per chunk encode (ckks.cpp:263-307) + encrypt (ckks.cpp:350-379). The
// reference's Sampler stream (mt19937_64, sampling.cpp) is sequential, so the
// draws -- the sparse ternary r, the CBD errors e0, e1 -- and the encoding FFT
// stay on the host (engine.cu); the device lifts the small integers and the
// rounded message into every limb, runs the forward NTTs and forms
//   c0 = p0 * r + e0 + m,   c1 = p1 * r + e1   (evaluation domain),
// word-identical to the reference for the same Sampler state.
#pragma once

#include "common.cuh"

namespace lcl {

// ws[c][poly][i][a] for poly = (m, r, e0, e1): the signed integers of chunk c
// reduced into [0, q_i). rounded: [C][N] int64 (|v| < 4.6e18), small:
// [C][3][N] int8 (r, e0, e1).
__global__ void __launch_bounds__(256)
    encrypt_lift(const long long* __restrict__ rounded, const signed char* __restrict__ small,
                 u32 C, u32 m, u32 logn, u64* __restrict__ ws,
                 const PrimeConst* __restrict__ primes) {
  const u64 N = 1ull << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)C * m * N) return;
  const u64 c = gid / (m * N);
  const u64 rem = gid - c * m * N;
  const u32 i = (u32)(rem >> logn);
  const u64 a = rem & (N - 1);
  const PrimeConst P = primes[i];
  const u64 q = P.q;
  u64* w = ws + c * 4 * m * N + (u64)i * N + a;
  const long long v = rounded[c * N + a];
  const u64 mag = reduce64((u64)(v < 0 ? -v : v), P);
  w[0] = v < 0 ? (mag == 0 ? 0 : q - mag) : mag;  // ckks.cpp:297-303
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int s = small[(c * 3 + k) * N + a];
    w[(u64)(k + 1) * m * N] = s >= 0 ? (u64)s : q - (u64)(-s);  // set_coeff, sampling.cpp
  }
}

// out[c][x][i][a]: c0 = p0 r + e0 + m, c1 = p1 r + e1 over the transformed ws.
__global__ void __launch_bounds__(256)
    encrypt_combine(const u64* __restrict__ ws, const u64* __restrict__ pk, u32 C, u32 m,
                    u32 logn, u64* __restrict__ out, const PrimeConst* __restrict__ primes) {
  const u64 N = 1ull << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)C * m * N) return;
  const u64 c = gid / (m * N);
  const u64 rem = gid - c * m * N;
  const u32 i = (u32)(rem >> logn);
  const PrimeConst P = primes[i];
  const u64 q = P.q;
  const u64* w = ws + c * 4 * m * N + rem;
  const u64 mm = w[0], r = w[m * N], e0 = w[2 * m * N], e1 = w[3 * m * N];
  u64* o = out + c * 2 * m * N + rem;
  o[0] = add_mod(add_mod(mul_mod(__ldg(pk + rem), r, P), e0, q), mm, q);
  o[m * N] = add_mod(mul_mod(__ldg(pk + m * N + rem), r, P), e1, q);
}

}  // namespace lcl
