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

// ---- key generation (ckks.cpp:195-261)
// rows [R][N] of small signed integers (one value per coefficient, every row)
// reduced into the row primes; prime of row r = prime_of(r).
__global__ void __launch_bounds__(256)
    lift_small(const signed char* __restrict__ small, u32 rows, u32 logn, u32 full,
               u64* __restrict__ out, const PrimeConst* __restrict__ primes) {
  const u64 N = 1ull << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)rows * N) return;
  const u32 r = (u32)(gid >> logn);
  const u64 q = primes[r <= full ? r : full].q;
  const int v = small[gid & (N - 1)];
  out[gid] = v >= 0 ? (u64)v : q - (u64)(-v);
}

// k0 = -a s + e over rows [R][N] (row r uses prime r; the special prime is
// the last row); with target: row j also += theta_j * target_j,
// theta_j = P mod q_j (make_switch_key, ckks.cpp:204-222).
__global__ void __launch_bounds__(256)
    key_rows(const u64* __restrict__ a, const u64* __restrict__ sk, const u64* __restrict__ e,
             u32 rows, u32 logn, const u64* __restrict__ target, u32 j, u64 theta,
             u64* __restrict__ k0, const PrimeConst* __restrict__ primes) {
  const u64 N = 1ull << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)rows * N) return;
  const u32 r = (u32)(gid >> logn);
  const PrimeConst P = primes[r];
  const u64 q = P.q;
  const u64 as = mul_mod(a[gid], sk[gid], P);
  u64 v = add_mod(as ? q - as : 0, e[gid], q);
  if (target && r == j) v = add_mod(v, mul_mod(target[gid], theta, P), q);
  k0[gid] = v;
}

// out[r][i] = in[r][perm[i]] (apply_galois in the evaluation domain, rns.cpp:534-547)
__global__ void __launch_bounds__(256)
    permute_rows(const u64* __restrict__ in, const u32* __restrict__ perm, u32 rows, u32 logn,
                 u64* __restrict__ out) {
  const u64 N = 1ull << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)rows * N) return;
  const u64 r = gid >> logn;
  out[gid] = in[(r << logn) + __ldg(perm + (gid & (N - 1)))];
}

// out = x * y pointwise over rows [R][N] (s^2 for the relinearization key)
__global__ void __launch_bounds__(256)
    square_rows(const u64* __restrict__ x, u32 rows, u32 logn, u64* __restrict__ out,
                const PrimeConst* __restrict__ primes) {
  const u64 N = 1ull << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)rows * N) return;
  out[gid] = mul_mod(x[gid], x[gid], primes[(u32)(gid >> logn)]);
}

}  // namespace lcl
