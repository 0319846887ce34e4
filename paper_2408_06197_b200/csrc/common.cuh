// Shared device arithmetic for the Lancelot server path on sm_100a.
//
// All residues are u64 in [0, q) at every observable boundary; inside kernels
// values may be kept lazily in [0, 2q) or [0, 4q) (Harvey butterflies). Every
// prime of the chain is < 2^55 (q0 44 bits, scale primes 40 bits, special 54
// bits: CkksParams defaults, reference ckks.hpp:39-55), so 4q < 2^57 never
// overflows a word. Results are bit-identical to the reference because the
// arithmetic is exact modular arithmetic: any evaluation order yields the same
// fully reduced residue.
#pragma once

#include <cstdint>

typedef uint64_t u64;
typedef unsigned int u32;
typedef uint8_t u8;

#define LCL_MAXP 16  // q primes + special supported by one context

// Per-prime constants, resident in __constant__ memory of every module.
struct PrimeConst {
  u64 q;
  u64 two_q;
  u64 ratio_lo, ratio_hi;  // floor((2^128 - 1) / q): exact 128-bit Barrett (modmath.hpp:62-73)
  u64 one_shoup;           // floor(2^64 / q): 64-bit reduction via Shoup with w = 1
  u64 half;                // q >> 1: centred-lift threshold (rns.cpp:370-378)
  u64 n_inv, n_inv_shoup;  // N^-1 mod q
  u64 w1n, w1n_shoup;      // iroot[1] * N^-1: last inverse stage with the scaling folded in
  u32 mu56;                // floor(2^56 / q): 32x32 Barrett quotient for lifts (v < 2^55)
  u32 mu62;                // floor(2^62 / q): reduce62 for lazy NTT outputs (x < 2^62)
  // FP64-pipe companions (used only for primes below 2^46, see "FP64 residue
  // arithmetic" below): q, 1/q, and (w, w/q) for the N^-1 scalings.
  double qf, qinvf;
  double ninvf, ninvq;
  double w1nf, w1nq;
};

// Twiddle / constant tables of a context, passed by value to every NTT kernel.
// fp_mask bit p set: rows of prime p run their butterflies on the FP64 pipe.
struct NttTabs {
  const ulonglong2* tw;   // (psi^brv, Shoup) per prime
  const ulonglong2* itw;  // inverse table
  const double2* twf;     // (psi^brv, psi^brv / q) as doubles
  const double2* itwf;
  const PrimeConst* primes;
  // Block-pass twiddles re-ordered per 256-point block (two-pass rings):
  // btw[p][b][pos], pos = blk_tw_pos(lm, g, l), so the 16 lanes of a block
  // read 16 consecutive entries at every stage (see ntt.cuh GlobalTw).
  const ulonglong2* btw;
  const ulonglong2* bitw;
  const double2* btwf;
  const double2* bitwf;
  u32 fp_mask;
  u32 logn;
};

// Row addressing for batched transforms. Row r of a launch is row
// sub = r % rows_per_item of item = r / rows_per_item; items come in groups of
// items_per_group (e.g. the (c0, c1) halves of one ciphertext):
//   base + (item / ipg) * group_stride + (item % ipg) * item_stride + sub * row_stride
// and uses prime prime_of[sub].
struct RowMap {
  u64* base;
  u64 group_stride;
  u64 item_stride;
  u64 row_stride;
  u32 rows_per_item;
  u32 items_per_group;
  unsigned char prime_of[LCL_MAXP * 2];
};

__device__ __forceinline__ u64* row_ptr(const RowMap& m, u32 r) {
  const u32 item = r / m.rows_per_item;
  const u32 sub = r - item * m.rows_per_item;
  const u32 g = item / m.items_per_group;
  const u32 h = item - g * m.items_per_group;
  return m.base + (u64)g * m.group_stride + (u64)h * m.item_stride + (u64)sub * m.row_stride;
}
__device__ __forceinline__ u32 row_prime(const RowMap& m, u32 r) {
  return m.prime_of[r % m.rows_per_item];
}

// ---------------------------------------------------------------- scalar ops
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) {
  u64 s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) {
  return a >= b ? a - b : a + q - b;
}
__device__ __forceinline__ u64 csub(u64 a, u64 q) { return a >= q ? a - q : a; }

// Shoup product a*w mod q for fixed w with ws = floor(w * 2^64 / q).
// Any a < 2^64 is accepted; the result lies in [0, 2q).
__device__ __forceinline__ u64 mul_shoup_lazy(u64 a, u64 w, u64 ws, u64 q) {
  const u64 hi = __umul64hi(a, ws);
  return a * w - hi * q;
}
// Shoup product with a truncated quotient: the y0*s0 partial product and the
// carries out of the two 32x32 cross products are dropped, so the quotient
// estimate is at most 3 below floor(a*w/q) and the result lies in [0, 4q).
// Three IMAD.WIDE instead of four plus their carry chain.
__device__ __forceinline__ u64 mul_shoup_lazy4(u64 a, u64 w, u64 ws, u64 q) {
  const u32 a0 = (u32)a, a1 = (u32)(a >> 32);
  const u32 s0 = (u32)ws, s1 = (u32)(ws >> 32);
  const u64 t1 = (u64)a1 * s0, t2 = (u64)a0 * s1;
  const u64 hi = (u64)a1 * s1 + (t1 >> 32) + (t2 >> 32);
  return a * w - hi * q;
}
__device__ __forceinline__ u64 mul_shoup(u64 a, u64 w, u64 ws, u64 q) {
  return csub(mul_shoup_lazy(a, w, ws, q), q);
}
// a mod q for any 64-bit a.
__device__ __forceinline__ u64 reduce64(u64 a, const PrimeConst& p) {
  return csub(a - __umul64hi(a, p.one_shoup) * p.q, p.q);
}

// Exact x mod q for a lazy word x < 2^62 (2^39 < q < 2^55): one 32x32 high
// product estimates the quotient (qh = floor(x/q) - {0,1,2}), the remainder
// x - qh q lies in [0, 3q) and two conditional subtractions finish. Costs one
// IMAD.HI + one IMAD.WIDE instead of reduce64's full 64x64 high product
// (IMAD.WIDE / IMAD.HI retire at half the rate of IMAD on sm_100).
__device__ __forceinline__ u64 reduce62(u64 x, u64 q, u32 mu62) {
  const u32 qh = __umulhi((u32)(x >> 30), mu62);
  u64 r = x - (u64)qh * q;
  r = r >= q ? r - q : r;
  return r >= q ? r - q : r;
}

// ------------------------------------------------ FP64 residue arithmetic
// B200 keeps a full-rate FP64 pipe (64 DFMA/clk/SM, measured) beside the
// integer pipes, and an FP64 butterfly on integer-valued doubles retires 2.3x
// faster than the 64-bit integer (Shoup) butterfly
// (tools/microbench/fp64_pipe.cu). For a prime q < 2^46 a residue is held as
// an exact integer-valued double in signed lazy form; every operation below
// is exact (no rounding ever reaches the integer result), so the fully
// reduced outputs are the reference's words.
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: round-to-integer bias
constexpr double kTwo52 = 4503599627370496.0;
constexpr long long kMagicBits = 0x4338000000000000ll;

// y * w mod q in signed lazy form, |result| <= 0.75 q, for integers |y| <= 2^51,
// 0 <= w < q < 2^46 and wq = fl(w / q). ph + pl = y*w exactly (FMA two-product);
// qt = round(y * wq) is within 0.75 of y*w/q, so ph - qt*q and the final sum
// are integers below 2^47 and both roundings are exact.
__device__ __forceinline__ double f_mulmod(double y, double w, double wq, double q) {
  const double ph = __dmul_rn(y, w);
  const double pl = __fma_rn(y, w, -ph);
  const double qt = __dadd_rn(__fma_rn(y, wq, kMagic), -kMagic);
  return __dadd_rn(__fma_rn(-qt, q, ph), pl);
}
// x - q * round(x / q) for an integer |x| <= 2^51: |result| <= 0.75 q. For
// |x| <= 0.75 q the quotient is exact and the result is the centred residue in
// [-(q-1)/2, (q-1)/2] (q odd: no ties) -- the reference's centred lift
// (rns.cpp:370-378, v > q/2 means v - q).
__device__ __forceinline__ double f_reduce(double x, double q, double qinv) {
  const double qt = __dadd_rn(__fma_rn(x, qinv, kMagic), -kMagic);
  return __fma_rn(-qt, q, x);
}
// u64 x < 2^52 -> exact double.
__device__ __forceinline__ double u2d(u64 x) {
  return __dadd_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), -kTwo52);
}
// integer-valued |r| < 2^51 -> int64.
__device__ __forceinline__ long long d2ll(double r) {
  return __double_as_longlong(__dadd_rn(r, kMagic)) - kMagicBits;
}
// lazy |x| <= 2^51 -> fully reduced u64 in [0, q).
__device__ __forceinline__ u64 d_canon(double x, double q, double qinv, u64 qi) {
  const long long i = d2ll(f_reduce(x, q, qinv));
  return (u64)(i + ((i >> 63) & (long long)qi));
}

// Exact reduction of the 128-bit value (hi, lo) mod q (modmath.hpp:62-73).
__device__ __forceinline__ u64 reduce128(u64 lo, u64 hi, const PrimeConst& p) {
  // q_hat = floor(x * ratio / 2^128), computed from the three upper partial
  // products exactly as the reference does, in 64-bit halves.
  const u64 c0_hi = __umul64hi(lo, p.ratio_lo);
  const u64 c1_lo = lo * p.ratio_hi;
  const u64 c1_hi = __umul64hi(lo, p.ratio_hi);
  // c1 = lo*rhi + c0_hi  (128-bit)
  const u64 c1l = c1_lo + c0_hi;
  const u64 c1h = c1_hi + (c1l < c1_lo ? 1ull : 0ull);
  // c2 = hi*rlo + c1l   (only the high word is needed)
  const u64 c2_lo = hi * p.ratio_lo;
  const u64 c2_hi = __umul64hi(hi, p.ratio_lo);
  const u64 c2l = c2_lo + c1l;
  const u64 c2h = c2_hi + (c2l < c2_lo ? 1ull : 0ull);
  const u64 q_hat = hi * p.ratio_hi + c1h + c2h;
  return csub(lo - q_hat * p.q, p.q);
}

__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, const PrimeConst& p) {
  return reduce128(a * b, __umul64hi(a, b), p);
}

// 128-bit accumulate (lo, hi) += a * b.
__device__ __forceinline__ void mac128(u64& lo, u64& hi, u64 a, u64 b) {
  asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\tmadc.hi.u64 %1, %2, %3, %1;"
      : "+l"(lo), "+l"(hi)
      : "l"(a), "l"(b));
}

// ------------------------------------------------ split-23 product sums
// Operands below 2^46 are split into 23-bit halves x = x1*2^23 + x0. A product
// then needs four 32x32->64 multiply-adds into three 64-bit partial sums
//   s0 += x0*y0, s1 += x0*y1 + x1*y0, s2 += x1*y1     (each term < 2^47)
// that cannot overflow for fewer than 2^16 accumulated products. The value
// is s0 + s1*2^23 + s2*2^46 and is reduced once at the end.
struct Split {
  u32 lo, hi;
};
__device__ __forceinline__ Split split23(u64 x) {
  Split s;
  s.lo = (u32)x & 0x7FFFFFu;
  s.hi = (u32)(x >> 23);
  return s;
}
__device__ __forceinline__ u64 wmul(u32 a, u32 b) { return (u64)a * (u64)b; }

// acc += a * b with one IMAD.WIDE.U32 (64-bit accumulate form).
__device__ __forceinline__ void madw(u64& acc, u32 a, u32 b) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

struct Acc3 {
  u64 s0, s1, s2;
  __device__ __forceinline__ void zero() { s0 = s1 = s2 = 0; }
  __device__ __forceinline__ void mac(Split x, Split y) {
    madw(s0, x.lo, y.lo);
    madw(s1, x.lo, y.hi);
    madw(s1, x.hi, y.lo);
    madw(s2, x.hi, y.hi);
  }
  __device__ __forceinline__ void sq(Split x) {  // x^2: the cross term as lo * (2 hi)
    madw(s0, x.lo, x.lo);
    madw(s1, x.lo, x.hi << 1);  // x.hi < 2^23, so 2 x.hi fits 32 bits
    madw(s2, x.hi, x.hi);
  }
  // x^2 with the cross term halved: s1 += lo * hi (value = s0 + s1*2^24 + s2*2^46,
  // see reduce_sq); one IMAD.WIDE and no shift per square.
  __device__ __forceinline__ void sqh(Split x) {
    madw(s0, x.lo, x.lo);
    madw(s1, x.lo, x.hi);
    madw(s2, x.hi, x.hi);
  }
  // Fully reduced value mod q.
  __device__ __forceinline__ u64 reduce(const PrimeConst& p) const { return reduce_sh<23>(p); }
  __device__ __forceinline__ u64 reduce_sq(const PrimeConst& p) const { return reduce_sh<24>(p); }
  template <int SH>
  __device__ __forceinline__ u64 reduce_sh(const PrimeConst& p) const {
    // v = s0 + s1*2^SH + s2*2^46 as a 128-bit (lo, hi).
    u64 lo = s0, hi = 0;
    const u64 a = s1 << SH, ah = s1 >> (64 - SH);
    lo += a;
    hi += ah + (lo < a ? 1ull : 0ull);
    const u64 b = s2 << 46, bh = s2 >> 18;
    lo += b;
    hi += bh + (lo < b ? 1ull : 0ull);
    return reduce128(lo, hi, p);
  }
};

// ------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, no tensor map: contiguous byte ranges) with
// mbarrier completion, and L2 bulk prefetch (sm_90+ PTX; SASS UBLKCP, SYNCS).
__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses of shared memory ordered before later async-proxy
// (TMA) writes to it
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, u32 bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
