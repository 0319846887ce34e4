// KGC side of a round: batched decryption and decoding of the
// server's outputs on the device, word- and bit-identical to the reference's
// CkksContext::decrypt_values (ckks.cpp:381-393) = decode(decrypt(ct, sk)):
//   decrypt   m = c1 * s + c0 per limb (evaluation domain)      ckks.cpp:381-388
//   decode    inverse NTT, then the 2-prime CRT lift of limbs 0 and 1 to a
//             signed coefficient / scale (one prime: the centred residue),
//                                                               ckks.cpp:313-348
//             then Embedding::coeffs_to_slots: twist, radix-2 DIT FFT with
//             the positive-exponent roots, real part at slot_index
//                                                               encoding.cpp:90-134
// Every double operation mirrors the reference's (x86-64 build without FMA
// contraction, std::complex<double> products as (ac - bd, ad + bc)), with
// explicit round-to-nearest intrinsics so nvcc cannot contract them, so the
// decoded values are the reference's bit for bit.
#pragma once

#include "common.cuh"

namespace lcl {

// m[b][i][a] = c1 * s + c0 (mod q_i); ct [B][2][m][N], sk rows [m][N].
__global__ void __launch_bounds__(256)
    decrypt_rows(const u64* __restrict__ ct, const u64* __restrict__ sk, u32 B, u32 m, u32 logn,
                 u64* __restrict__ out, const PrimeConst* __restrict__ primes) {
  const u64 slots = (u64)m << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)B * slots) return;
  const u64 b = gid / slots, s = gid - b * slots;
  const PrimeConst P = primes[(u32)(s >> logn)];
  const u64* c = ct + b * 2 * slots;
  out[gid] = add_mod(mul_mod(c[slots + s], __ldg(sk + s), P), c[s], P.q);
}

// Correctly rounded conversion of x < 2^128 to double (the reference's
// static_cast<double>(unsigned __int128)).
__device__ __forceinline__ double u128_to_double(u64 lo, u64 hi) {
  if (hi == 0) return __ull2double_rn(lo);
  const int sh = 64 - __clzll(hi);  // significant bits of hi
  if (sh == 64) return ldexp(__ull2double_rn(hi | (lo != 0 ? 1ull : 0ull)), 64);
  const u64 top = (hi << (64 - sh)) | (lo >> sh);
  const u64 sticky = (lo << (64 - sh)) != 0 ? 1ull : 0ull;  // bits shifted out
  return ldexp(__ull2double_rn(top | sticky), sh);  // sticky sits 11 bits below the rounding bit
}

__device__ __forceinline__ double2 cmul(double2 a, double2 w) {  // (ac - bd, ad + bc)
  return make_double2(__dsub_rn(__dmul_rn(a.x, w.x), __dmul_rn(a.y, w.y)),
                      __dadd_rn(__dmul_rn(a.x, w.y), __dmul_rn(a.y, w.x)));
}

// Coefficient rows (after the inverse NTT) -> twisted FFT input in
// bit-reversed position: buckets[b][brv(i)] = (coeff(i), coeff(i + h)) * twist[i].
// crt = {q0, q1, inv01 = q0^-1 mod q1, its Shoup word}; count = live limbs.
struct CrtConst {
  u64 q0, q1, inv01, inv01s;
};
__device__ __forceinline__ double crt_coeff(const u64* rows, u64 n, u64 i, u32 count,
                                           const CrtConst& k, double scale) {
  double c;
  if (count >= 2) {
    const u64 r0 = rows[i];
    const u64 r0m = r0 >= k.q1 ? r0 % k.q1 : r0;
    const u64 diff = sub_mod(rows[n + i], r0m, k.q1);
    const u64 t = mul_shoup(diff, k.inv01, k.inv01s, k.q1);
    // x = q0 * t + r0 (u128), q01 = q0 * q1, half = q01 >> 1
    u64 xlo = k.q0 * t, xhi = __umul64hi(k.q0, t);
    xlo += r0;
    xhi += xlo < r0 ? 1 : 0;
    const u64 qlo = k.q0 * k.q1, qhi = __umul64hi(k.q0, k.q1);
    const u64 hlo = (qlo >> 1) | (qhi << 63), hhi = qhi >> 1;
    const bool neg = xhi > hhi || (xhi == hhi && xlo > hlo);
    if (neg) {
      const u64 dlo = qlo - xlo, dhi = qhi - xhi - (qlo < xlo ? 1 : 0);
      c = -u128_to_double(dlo, dhi);
    } else {
      c = u128_to_double(xlo, xhi);
    }
  } else {
    const u64 r = rows[i], half = k.q0 >> 1;
    c = r > half ? -__ull2double_rn(k.q0 - r) : __ull2double_rn(r);
  }
  return __ddiv_rn(c, scale);
}

__global__ void __launch_bounds__(256)
    decode_twist(const u64* __restrict__ coef, u32 B, u32 count, u32 logn, CrtConst k,
                 double scale, const double2* __restrict__ twist, const u32* __restrict__ brv,
                 double2* __restrict__ buckets) {
  const u32 h = 1u << (logn - 1);
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)B * h) return;
  const u64 b = gid / h;
  const u32 i = (u32)(gid - b * h);
  const u64 n = 1ull << logn;
  const u64* rows = coef + b * count * n;
  const double2 v = make_double2(crt_coeff(rows, n, i, count, k, scale),
                                 crt_coeff(rows, n, i + h, count, k, scale));
  buckets[b * h + __ldg(brv + i)] = cmul(v, __ldg(twist + i));
}

// Radix-2 DIT stages len = 2 .. min(h, 256) inside 256-point blocks (after
// the bit-reversal): butterfly (u, u + len/2) with roots[k * h / len].
__global__ void __launch_bounds__(128)
    fft_blocks(double2* __restrict__ a, u32 logh, const double2* __restrict__ roots) {
  __shared__ double2 s[256];
  const u32 h = 1u << logh;
  const u32 bs = h < 256 ? h : 256;
  double2* blk = a + (u64)blockIdx.x * bs;
  for (u32 e = threadIdx.x; e < bs; e += blockDim.x) s[e] = blk[e];
  __syncthreads();
  for (u32 len = 2; len <= bs; len <<= 1) {
    const u32 hl = len >> 1;
    for (u32 t = threadIdx.x; t < bs / 2; t += blockDim.x) {
      const u32 k = t % hl, u = (t / hl) * len + k;
      const double2 w = __ldg(roots + (u64)k * (h / len));
      const double2 x = s[u], v = cmul(s[u + hl], w);
      s[u] = make_double2(__dadd_rn(x.x, v.x), __dadd_rn(x.y, v.y));
      s[u + hl] = make_double2(__dsub_rn(x.x, v.x), __dsub_rn(x.y, v.y));
    }
    __syncthreads();
  }
  for (u32 e = threadIdx.x; e < bs; e += blockDim.x) blk[e] = s[e];
}

// Stages len = 512 .. h: element e = t * 256 + j; every butterfly stays in
// column j. A CTA owns 16 columns x h/256 rows of one transform in shared
// memory (dynamic: h / 256 * 16 complex).
__global__ void __launch_bounds__(256)
    fft_columns(double2* __restrict__ a, u32 logh, const double2* __restrict__ roots) {
  extern __shared__ double2 sc[];  // [rows][16]
  const u32 h = 1u << logh, rows = h >> 8;
  const u32 groups = 16;  // 256 columns / 16 per CTA
  const u64 b = blockIdx.x / groups;
  const u32 j0 = (blockIdx.x % groups) * 16;
  double2* base = a + b * h;
  for (u32 e = threadIdx.x; e < rows * 16; e += blockDim.x) {
    const u32 t = e >> 4, jj = e & 15;
    sc[e] = base[(u64)t * 256 + j0 + jj];
  }
  __syncthreads();
  for (u32 len = 512; len <= h; len <<= 1) {
    const u32 hr = len >> 9;  // half length in rows
    for (u32 f = threadIdx.x; f < rows * 8; f += blockDim.x) {
      const u32 jj = f & 15, bt = f >> 4;            // butterfly row index
      const u32 tu = (bt / hr) * (2 * hr) + bt % hr;  // row of u
      const u32 k = (tu % (2 * hr)) * 256 + j0 + jj;  // offset inside its group
      const double2 w = __ldg(roots + (u64)k * (h / len));
      const u32 iu = tu * 16 + jj, iv = (tu + hr) * 16 + jj;
      const double2 x = sc[iu], v = cmul(sc[iv], w);
      sc[iu] = make_double2(__dadd_rn(x.x, v.x), __dadd_rn(x.y, v.y));
      sc[iv] = make_double2(__dsub_rn(x.x, v.x), __dsub_rn(x.y, v.y));
    }
    __syncthreads();
  }
  for (u32 e = threadIdx.x; e < rows * 16; e += blockDim.x) {
    const u32 t = e >> 4, jj = e & 15;
    base[(u64)t * 256 + j0 + jj] = sc[e];
  }
}

// slots[b][j] = buckets[b][slot_index[j]].re
__global__ void __launch_bounds__(256)
    decode_slots(const double2* __restrict__ buckets, u32 B, u32 logh,
                 const u32* __restrict__ slot_index, double* __restrict__ out) {
  const u32 h = 1u << logh;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)B * h) return;
  const u64 b = gid >> logh;
  out[gid] = buckets[b * h + __ldg(slot_index + (gid & (h - 1)))].x;
}

// KGC distance entries (aggregation.cpp:232-258): the decrypted value of a
// matrix entry is slot 0 when the server reduced it, else the left-to-right
// sum of every slot (std::accumulate's order, round-to-nearest adds), then
// max(0, v / value_scale). One thread per entry.
__global__ void __launch_bounds__(128)
    entry_values(const double* __restrict__ slots, u32 B, u32 h, int reduced, double value_scale,
                 double* __restrict__ out) {
  const u32 b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* s = slots + (u64)b * h;
  double v = s[0];
  if (!reduced) {
    v = 0.0;
    for (u32 i = 0; i < h; ++i) v = __dadd_rn(v, s[i]);
  }
  out[b] = fmax(0.0, __ddiv_rn(v, value_scale));
}

}  // namespace lcl
