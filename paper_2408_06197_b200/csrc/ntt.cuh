// Negacyclic NTT over 64-bit primes for sm_100a.
//
// Mathematically identical to the reference transforms
// (proj/core/src/rns.cpp:140-181): forward = Cooley-Tukey with the
// bit-reversed psi-power table root[m + i] (natural order in, bit-reversed
// evaluation order out: index i holds a(psi^(2 brv(i) + 1))); inverse =
// Gentleman-Sande with the inverse table, then x N^-1. Because every output
// is fully reduced, the GPU factorisation below produces the same words.
//
// Factorisation for N = N1 * N2 (N2 = 256): element a = j + t*N2.
//   * The first log2(N1) CT stages pair rows t, t + N1/(2m) of each column j
//     with twiddle root[m + (t*m/N1)]: an N1-point NTT per column with the
//     table prefix root[1 .. N1-1]                        -> col pass
//   * The last log2(N2) stages stay inside block b = a / N2 and use
//     root[m'(N1 + b) + i'] at local stage m'              -> block pass
// The inverse runs the block pass first, then the column pass, fusing the
// N^-1 scaling into the column pass's store.
//
// Arithmetic: Harvey lazy butterflies. Forward values live in [0, 4q),
// inverse values in [0, 2q); twiddles are (w, floor(w 2^64 / q)) pairs.
// One HBM round trip per pass; shared memory only carries the transpose
// inside each pass. Loader / epilogue functors fuse the ModUp lift, the
// ModDown / rescale divide-and-round and the key-switch output adds into the
// first / last pass, so no standalone elementwise kernel touches HBM.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace lcl {

struct Tw {
  u64 w, ws;
};

__device__ __forceinline__ Tw ldtw(const ulonglong2* t, u32 idx) {
  const ulonglong2 v = __ldg(t + idx);
  return Tw{v.x, v.y};
}

// Forward CT butterfly without intermediate reduction: with t = y*w mod q in
// [0, 4q) (truncated Shoup quotient), x' = x + t and y' = x + 4q - t both stay
// below B + 4q when x < B. Starting from inputs < q, after s stages every
// value is < (1 + 4s) q; for s <= 17 and q < 2^55 that is < 69 * 2^55 < 2^62,
// so no word overflows and the only reduction is the final one (reduce62).
// The Shoup product accepts any y < 2^64. (two_q carries 4q here.)
__device__ __forceinline__ void ct_bfly(u64& x, u64& y, Tw w, u64 q, u64 four_q) {
  const u64 t = mul_shoup_lazy4(y, w.w, w.ws, q);
  const u64 a = x;
  x = a + t;
  y = a + (four_q - t);
}

// Inverse GS butterfly: x, y in [0, 2q) -> x', y' in [0, 2q).
__device__ __forceinline__ void gs_bfly(u64& x, u64& y, Tw w, u64 q, u64 two_q) {
  const u64 a = x, b = y;
  const u64 s = a + b;
  x = s >= two_q ? s - two_q : s;
  y = mul_shoup_lazy(a - b + two_q, w.w, w.ws, q);
}

// Padded shared-memory slot of block element i (bank-conflict-free for both
// the l + 16 e and the 16 l + e access patterns).
__device__ __forceinline__ u32 pad16(u32 i) { return i + (i >> 4); }

// ------------------------------------------------------------ loaders
// A loader is bound once per row (all address / constant lookups hoisted):
//   auto row = ld.bind(r, dst_prime_index, dst);  row(a) -> value < q
struct PlainLoad {
  RowMap in;
  struct Row {
    const u64* p;
    __device__ __forceinline__ u64 operator()(u32 a) const { return __ldg(p + a); }
  };
  __device__ __forceinline__ Row bind(u32 r, u32, const PrimeConst&) const {
    return Row{row_ptr(in, r)};
  }
  __host__ __device__ static constexpr double rows_read(double rows, u32) { return rows; }
};

// Centred lift of a coefficient-domain source row into the destination prime
// (single-prime mod_up branch, rns.cpp:367-383; the lift inside
// divide_and_round_by_last, rns.cpp:484-494). Destination row r of a launch
// reads source row (r / rows_per_item) * (rows_per_item / fan) + (r % rows_per_item) / fan.
//
// v mod q_d uses a 32x32 Barrett quotient: with v < 2^55 and 2^39 < q_d <
// 2^55, qh = ((v >> 24) * floor(2^56 / q_d)) >> 32 is floor(v / q_d) or one
// less, so v - qh q_d lies in [0, 2 q_d); the centring correction adds
// q_d - (q_s mod q_d). The value handed to the forward NTT is therefore
// congruent to the reference's lift and lies in [0, 3 q_d), which the
// reduction-free butterflies absorb ((3 + 4 s) q_d < 2^62 for s <= 17).
// With SIGMA the source is read through the Galois automorphism X -> X^elt in
// the coefficient domain (entry = src index | negate << 31); lifting commutes
// with that signed permutation (small rings only; the two-pass rings apply the
// permutation block-locally in the evaluation domain).
template <bool SIGMA>
struct LiftLoadT {
  RowMap src;
  u32 rows_per_item;
  u32 fan;
  u32 nprimes;               // full + 1
  const PrimeConst* primes;  // device table
  const u64* smod;           // smod[s * nprimes + d] = q_s mod q_d
  const u32* sigma;          // SIGMA only
  struct Row {
    const u64* s;
    const u32* sigma;
    u64 qs, half, corr, q;
    u32 mu;
    __device__ __forceinline__ u64 operator()(u32 a) const {
      u64 v;
      if (SIGMA) {
        const u32 e = __ldg(sigma + a);
        v = __ldg(s + (e & 0x7FFFFFFFu));
        if ((e >> 31) && v) v = qs - v;
      } else {
        v = __ldg(s + a);
      }
      const u64 qh = ((u64)(u32)(v >> 24) * mu) >> 32;
      u64 x = v - qh * q;
      if (v > half) x += corr;
      return x;
    }
  };
  __device__ __forceinline__ Row bind(u32 r, u32 dpi, const PrimeConst& dst) const {
    const u32 item = r / rows_per_item;
    const u32 sub = (r - item * rows_per_item) / fan;
    const u32 srow = item * (rows_per_item / fan) + sub;
    const u32 sp = row_prime(src, srow);
    Row w;
    w.s = row_ptr(src, srow);
    w.sigma = sigma;
    w.qs = __ldg(&primes[sp].q);
    w.half = __ldg(&primes[sp].half);
    w.corr = dst.q - __ldg(smod + sp * nprimes + dpi);
    w.q = dst.q;
    w.mu = dst.mu56;
    return w;
  }
};
using LiftLoad = LiftLoadT<false>;
using LiftSigmaLoad = LiftLoadT<true>;

// ------------------------------------------------------------ epilogues
// auto row = epi.bind(r, dst_prime_index, dst);  row(a, value < q)
struct PlainStore {
  static constexpr bool kNeedsReduced = true;
  RowMap out;
  struct Pre {};
  struct Row {
    u64* p;
    __device__ __forceinline__ void operator()(u32 a, u64 v) const { p[a] = v; }
    __device__ __forceinline__ void stage(u64*, u32, u32) const {}
    __device__ __forceinline__ void prefetch(Pre&, u32, const u64*) const {}
    __device__ __forceinline__ void store(const Pre&, u32 a, u64 v) const { p[a] = v; }
  };
  __device__ __forceinline__ Row bind(u32 r, u32, const PrimeConst&) const {
    return Row{row_ptr(out, r)};
  }
};

// Divide-and-round output (rns.cpp:496-505) fused with the key-switch output
// additions:  out = (x - lift) * p^-1  [+ add1[a]]  [+ add2[perm[a]] on the
// first item of every group, i.e. the c0 half]. add2 must not alias out
// (gathered reads); add1 may alias out (same thread reads then writes one word).
struct DivRoundStore {
  static constexpr bool kNeedsReduced = false;  // the lift may be any lazy word < 80q
  RowMap out;
  RowMap x;
  RowMap add1;  // base == nullptr: absent
  RowMap add2;  // base == nullptr: absent
  const u32* perm;  // gather for add2 (nullptr: identity)
  const ulonglong2* pinv;  // indexed by destination prime: (p^-1 mod q, shoup)
  struct Pre {
    u64 x, add;  // x[a] and the sum of the (up to two) addends
  };
  struct Row {
    u64* o;
    const u64* x;
    const u64* a1;
    const u64* a2;
    const u32* perm;
    u64 iv, ivs, q, q80;
    __device__ __forceinline__ void operator()(u32 a, u64 lift) const {
      Pre p;
      prefetch(p, a, nullptr);
      store(p, a, lift);
    }
    // With a permuted add2, the 256-element source block of block b is staged
    // into shared memory s first (block-local Galois permutation).
    __device__ __forceinline__ void stage(u64* s, u32 b, u32 l) const {
      if (a2 && perm) {
        const u32 src_blk = __ldg(perm + (b << 8)) >> 8;
#pragma unroll
        for (int e = 0; e < 16; ++e) s[pad16(l + 16 * e)] = a2[(src_blk << 8) + l + 16 * e];
        __syncwarp();
      }
    }
    __device__ __forceinline__ void prefetch(Pre& p, u32 a, const u64* s) const {
      p.x = x[a];
      u64 v = a1 ? a1[a] : 0;
      if (a2) {
        const u64 g = perm ? (s ? s[pad16(__ldg(perm + a) & 255u)] : a2[__ldg(perm + a)]) : a2[a];
        v = add_mod(v, g, q);
      }
      p.add = v;
    }
    __device__ __forceinline__ void store(const Pre& p, u32 a, u64 lift) const {
      // lift < 80q (lazy NTT output): x + 80q - lift > 0 and congruent
      const u64 v = mul_shoup(p.x + (q80 - lift), iv, ivs, q);
      o[a] = add_mod(v, p.add, q);
    }
  };
  __device__ __forceinline__ Row bind(u32 r, u32 dpi, const PrimeConst& P) const {
    Row w;
    const ulonglong2 iv = __ldg(pinv + dpi);
    w.o = row_ptr(out, r);
    w.x = row_ptr(x, r);
    w.a1 = add1.base ? row_ptr(add1, r) : nullptr;
    w.a2 = (add2.base && ((r / out.rows_per_item) % out.items_per_group) == 0) ? row_ptr(add2, r)
                                                                                : nullptr;
    w.perm = perm;
    w.iv = iv.x;
    w.ivs = iv.y;
    w.q = P.q;
    w.q80 = 80 * P.q;
    return w;
  }
};

// ------------------------------------------------------------ stage helpers
// Compile-time stage iteration: every register index below is a constant, so
// the 16/32-element tiles stay in registers (no local-memory arrays).
template <int I, int END, int STEP, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I != END) {
    f(std::integral_constant<int, I>{});
    static_for<I + STEP, END, STEP>(f);
  }
}

// One radix-2 stage over a register tile: groups of 2D consecutive elements,
// butterflies (g*2D + e, g*2D + e + D); twf(g) gives the group's twiddle.
template <int E, int D, class TwF>
__device__ __forceinline__ void ct_stage(u64 (&x)[E], const TwF& twf, u64 q, u64 two_q) {
  const u64 four_q = 2 * two_q;
#pragma unroll
  for (int g = 0; g < E / (2 * D); ++g) {
    const Tw w = twf(g);
#pragma unroll
    for (int e = 0; e < D; ++e) ct_bfly(x[g * 2 * D + e], x[g * 2 * D + e + D], w, q, four_q);
  }
}
template <int E, int D, class TwF>
__device__ __forceinline__ void gs_stage(u64 (&x)[E], const TwF& twf, u64 q, u64 two_q) {
#pragma unroll
  for (int g = 0; g < E / (2 * D); ++g) {
    const Tw w = twf(g);
#pragma unroll
    for (int e = 0; e < D; ++e) gs_bfly(x[g * 2 * D + e], x[g * 2 * D + e + D], w, q, two_q);
  }
}

// ------------------------------------------------------------ kernels
// Column pass, forward. CTA = 16 consecutive columns x N1 rows of one row-poly.
// Thread (c, k): column c, rows k + R e (phase 1, log2 E stages in registers),
// then rows k E + e (phase 2, log2 R stages) after one shared transpose.
template <int LOGN1, int E, class Loader>
__global__ void __launch_bounds__(16 * ((1 << LOGN1) / E))
    ntt_col_fwd(const __grid_constant__ RowMap out, const __grid_constant__ Loader ld,
                const ulonglong2* __restrict__ tw_all, const PrimeConst* __restrict__ primes,
                u32 logn) {
  constexpr int N1 = 1 << LOGN1;
  constexpr int R = N1 / E;
  constexpr int LOGE = __builtin_ctz(E);
  extern __shared__ u64 sm[];  // [N1][16]
  const u32 n = 1u << logn;
  const u32 n2 = n >> LOGN1;
  const u32 groups = n2 >> 4;
  const u32 r = blockIdx.x / groups;
  const u32 g = blockIdx.x - r * groups;
  const u32 c = threadIdx.x & 15, k = threadIdx.x >> 4;
  const u32 j = (g << 4) + c;
  const u32 pi = row_prime(out, r);
  const PrimeConst P = primes[pi];
  const ulonglong2* tw = tw_all + (u64)pi * n;
  u64 x[E];
  {
    const auto row = ld.bind(r, pi, P);
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = row(j + (k + R * e) * n2);
  }
  // phase 1: m = 1 .. E/2; group g of a stage is twiddle root[m + g]
  static_for<0, LOGE, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    ct_stage<E, (E >> (lm + 1))>(x, [&](int gi) { return ldtw(tw, (1 << lm) + gi); }, P.q, P.two_q);
  });
#pragma unroll
  for (int e = 0; e < E; ++e) sm[(k + R * e) * 16 + c] = x[e];
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = sm[(k * E + e) * 16 + c];
  // phase 2: m = E .. N1/2 on rows t = kE + e; distance N1/(2m) < R <= E
  static_for<LOGE, LOGN1, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = N1 >> (lm + 1);
    ct_stage<E, d>(x, [&](int gi) { return ldtw(tw, (1 << lm) + ((k * E + gi * 2 * d) >> (LOGN1 - lm))); },
                   P.q, P.two_q);
  });
  u64* o = row_ptr(out, r);
#pragma unroll
  for (int e = 0; e < E; ++e) o[j + (k * E + e) * n2] = x[e];
}

// Block pass body, forward: x[e] holds element l + 16 e of one 256-point
// block (coalesced order) on entry and the fully reduced output in the same
// order on exit. Phase 1 runs local stages m' = 1..8 on s = l + 16 e, phase 2
// m' = 16..128 on s = 16 l + e after a warp-local shared transpose.
template <int LOGN1, bool REDUCE = true>
__device__ __forceinline__ void blk_fwd_body(u64 (&x)[16], u64* s, const ulonglong2* tw, u32 b,
                                             u32 l, const PrimeConst& P) {
  constexpr int N1 = 1 << LOGN1;
  static_for<0, 4, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    ct_stage<16, (16 >> (lm + 1))>(x, [&](int gi) { return ldtw(tw, (N1 + b) * (1 << lm) + gi); },
                                   P.q, P.two_q);
  });
#pragma unroll
  for (int e = 0; e < 16; ++e) s[l + 16 * e + e] = x[e];
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = s[16 * l + e + l];
  static_for<4, 8, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = 256 >> (lm + 1);
    ct_stage<16, d>(x,
                    [&](int gi) { return ldtw(tw, (N1 + b) * (1 << lm) + ((16 * l + gi * 2 * d) >> (8 - lm))); },
                    P.q, P.two_q);
  });
  // REDUCE = false leaves the lazy words (< 71q, see ct_bfly) for consumers
  // that only feed them into a Shoup product, which accepts any 64-bit input.
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) s[16 * l + e + l] = REDUCE ? reduce62(x[e], P.q, P.mu62) : x[e];
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = s[l + 16 * e + e];
  __syncwarp();
}

// Block pass body, inverse: x[e] = element l + 16 e of block b (coalesced
// order, values < 2q) in and out; GS stages m' = 128 .. 1 (global m = N/2 .. N1).
template <int LOGN1>
__device__ __forceinline__ void blk_inv_body(u64 (&x)[16], u64* s, const ulonglong2* tw, u32 b,
                                             u32 l, const PrimeConst& P) {
  constexpr int N1 = 1 << LOGN1;
#pragma unroll
  for (int e = 0; e < 16; ++e) s[l + 16 * e + e] = x[e];
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = s[16 * l + e + l];
  static_for<7, 3, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = 256 >> (lm + 1);
    gs_stage<16, d>(x,
                    [&](int gi) { return ldtw(tw, (N1 + b) * (1 << lm) + ((16 * l + gi * 2 * d) >> (8 - lm))); },
                    P.q, P.two_q);
  });
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) s[16 * l + e + l] = x[e];
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = s[l + 16 * e + e];
  __syncwarp();
  static_for<3, -1, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    gs_stage<16, (16 >> (lm + 1))>(x, [&](int gi) { return ldtw(tw, (N1 + b) * (1 << lm) + gi); },
                                   P.q, P.two_q);
  });
}

// Galois permutation inside one 256-element block. In bit-reversed evaluation
// order the permutation maps every aligned output block onto exactly one
// input block (the low 8 index bits only touch the top 8 exponent bits), so a
// rotation's gather is a coalesced load of the source block followed by a
// shuffle through shared memory. src_blk = perm[blk * 256] >> 8.
__device__ __forceinline__ void block_gather(u64 (&x)[16], u64* s, const u64* src_block,
                                             const u32* perm, u32 blk, u32 l) {
#pragma unroll
  for (int e = 0; e < 16; ++e) s[pad16(l + 16 * e)] = __ldg(src_block + l + 16 * e);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = s[pad16(__ldg(perm + (blk << 8) + l + 16 * e) & 255u)];
  __syncwarp();
}

// Block pass, forward: 256-point blocks, 16 threads per block, 16 elements per
// thread, 4 blocks per CTA. The epilogue's operands are prefetched before the
// butterflies so their latency overlaps the arithmetic.
template <int LOGN1, class Epi>
__global__ void __launch_bounds__(64)
    ntt_blk_fwd(const __grid_constant__ RowMap in, const __grid_constant__ Epi epi,
                const ulonglong2* __restrict__ tw_all, const PrimeConst* __restrict__ primes,
                u32 logn) {
  constexpr int N1 = 1 << LOGN1;
  __shared__ u64 sm[4][256 + 16];
  const u32 n = 1u << logn;
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  const u32 blk_global = blockIdx.x * 4 + bw;
  const u32 r = blk_global / N1;
  const u32 b = blk_global - r * N1;
  const u32 pi = row_prime(in, r);
  const PrimeConst P = primes[pi];
  const ulonglong2* tw = tw_all + (u64)pi * n;
  const u64* src = row_ptr(in, r) + (b << 8);
  u64 x[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = src[l + 16 * e];
  blk_fwd_body<LOGN1, Epi::kNeedsReduced>(x, sm[bw], tw, b, l, P);
  const auto row = epi.bind(r, pi, P);
  row.stage(sm[bw], b, l);
  // operands of 4 elements in flight at a time: latency overlap without the
  // register cost of prefetching all 16
#pragma unroll
  for (int e0 = 0; e0 < 16; e0 += 4) {
    typename Epi::Pre pre[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) row.prefetch(pre[e], (b << 8) + l + 16 * (e0 + e), sm[bw]);
#pragma unroll
    for (int e = 0; e < 4; ++e) row.store(pre[e], (b << 8) + l + 16 * (e0 + e), x[e0 + e]);
  }
}

// ModUp block pass fused with the key inner product (ckks.cpp:464-518).
// A 16-thread group owns block blk of target row t of ciphertext b and walks
// the M digits: digit j is the column-pass output mid[b][j][t'] run through
// the block stages, except the identity row t == j, whose lifted NTT is the
// input limb itself (mod_up returns the row unchanged, rns.cpp:371-381), read
// through the rotation's evaluation-domain permutation when one is given.
// Each digit is multiplied by the key in Shoup form and accumulated lazily
// (< 4Mq), so the m(m+1) digit rows never reach HBM.
//   mid: [B][M][M][N] (t' = t < j ? t : t - 1); c1: limb j of item b at
//   c1 + b * c1_stride + j * N; key / key_shoup: [full][2][full+1][N];
//   acc: [B][2][M+1][N].
template <int LOGN1, int M>
__global__ void __launch_bounds__(64, 8)
    modup_ip_blk(u32 B, const u64* __restrict__ mid, const u64* __restrict__ c1, u64 c1_stride,
                 const u32* __restrict__ perm, const u64* __restrict__ key,
                 const u64* __restrict__ key_shoup, u32 full, u64* __restrict__ acc,
                 const ulonglong2* __restrict__ tw_all, const PrimeConst* __restrict__ primes,
                 u32 logn) {
  constexpr int N1 = 1 << LOGN1;
  __shared__ u64 sm[4][256 + 16];
  __shared__ u64 sacc[4][2][256];  // lazy accumulators (< 4Mq), coalesced order
  const u32 n = 1u << logn;
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  // the 4 groups of a CTA take 4 consecutive ciphertexts of the same
  // (target row, block): the key words they share are served from L1
  const u32 bq_count = (B + 3) >> 2;
  const u32 bq = blockIdx.x % bq_count;
  const u32 tb = blockIdx.x / bq_count;  // = t * N1 + blk
  const u32 t = tb / N1, blk = tb - t * N1;
  const u32 bi_raw = bq * 4 + bw;
  const bool live = bi_raw < B;
  const u32 bi = live ? bi_raw : B - 1;
  const u32 pi = t < (u32)M ? t : full;
  const PrimeConst P = primes[pi];
  const ulonglong2* tw = tw_all + (u64)pi * n;
  const u64 kstride = (u64)(full + 1) * n;
  const u32 a0 = (blk << 8) + l;
  u64* s0acc = sacc[bw][0];
  u64* s1acc = sacc[bw][1];
  // rotation: output block blk of every digit comes from block src_blk of the
  // unpermuted digit (block-local Galois permutation, see block_gather)
  const u32 src_blk = perm ? (__ldg(perm + (blk << 8)) >> 8) : blk;
#pragma unroll 1
  for (int j = 0; j < M; ++j) {
    u64 x[16];
    if (t == (u32)j) {
      const u64* src = c1 + (u64)bi * c1_stride + (u64)j * n + (src_blk << 8);
      if (perm) {
        block_gather(x, sm[bw], src, perm, blk, l);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = __ldg(src + l + 16 * e);
      }
    } else {
      const u32 tp = t < (u32)j ? t : t - 1;
      const u64* src = mid + (((u64)bi * M + j) * M + tp) * n + (src_blk << 8);
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = src[l + 16 * e];
      blk_fwd_body<LOGN1, false>(x, sm[bw], tw, src_blk, l, P);
      if (perm) {
        // the body left the (lazy) block in shared memory: permuted read
#pragma unroll
        for (int e = 0; e < 16; ++e)
          x[e] = sm[bw][pad16(__ldg(perm + (blk << 8) + l + 16 * e) & 255u)];
        __syncwarp();
      }
    }
    const u64* k0 = key + (2ull * j) * kstride + (u64)pi * n;
    const u64* k1 = k0 + kstride;
    const u64* ks0 = key_shoup + (2ull * j) * kstride + (u64)pi * n;
    const u64* ks1 = ks0 + kstride;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const u32 a = a0 + 16 * e;
      // each product < 4q: the M-term sums stay < 24q (M <= 6)
      const u64 p0 = mul_shoup_lazy4(x[e], __ldg(k0 + a), __ldg(ks0 + a), P.q);
      const u64 p1 = mul_shoup_lazy4(x[e], __ldg(k1 + a), __ldg(ks1 + a), P.q);
      const u32 si = l + 16 * e;
      s0acc[si] = j ? s0acc[si] + p0 : p0;
      s1acc[si] = j ? s1acc[si] + p1 : p1;
    }
  }
  if (!live) return;
  u64* o0 = acc + ((u64)bi * 2 * (M + 1) + t) * n;
  u64* o1 = o0 + (u64)(M + 1) * n;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const u32 si = l + 16 * e;
    o0[a0 + 16 * e] = reduce62(s0acc[si], P.q, P.mu62);
    o1[a0 + 16 * e] = reduce62(s1acc[si], P.q, P.mu62);
  }
}

// Block pass, inverse: GS stages m = N/2 .. N1 (local m' = 128 .. 1).
template <int LOGN1>
__global__ void __launch_bounds__(64)
    ntt_blk_inv(const __grid_constant__ RowMap in, const __grid_constant__ RowMap out,
                const ulonglong2* __restrict__ itw_all, const PrimeConst* __restrict__ primes,
                u32 logn) {
  constexpr int N1 = 1 << LOGN1;
  __shared__ u64 sm[4][256 + 16];
  const u32 n = 1u << logn;
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  const u32 blk_global = blockIdx.x * 4 + bw;
  const u32 r = blk_global / N1;
  const u32 b = blk_global - r * N1;
  const u32 pi = row_prime(in, r);
  const PrimeConst P = primes[pi];
  const ulonglong2* tw = itw_all + (u64)pi * n;
  const u64* src = row_ptr(in, r) + (b << 8);
  u64 x[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = src[l + 16 * e];
  blk_inv_body<LOGN1>(x, sm[bw], tw, b, l, P);
  u64* dst = row_ptr(out, r) + (b << 8);
#pragma unroll
  for (int e = 0; e < 16; ++e) dst[l + 16 * e] = x[e];
}

// Column pass, inverse: GS stages m = N1/2 .. 1, then x N^-1 and a full
// reduction; the result goes through the epilogue.
template <int LOGN1, int E, class Epi>
__global__ void __launch_bounds__(16 * ((1 << LOGN1) / E))
    ntt_col_inv(const __grid_constant__ RowMap in, const __grid_constant__ Epi epi,
                const ulonglong2* __restrict__ itw_all, const PrimeConst* __restrict__ primes,
                u32 logn) {
  constexpr int N1 = 1 << LOGN1;
  constexpr int R = N1 / E;
  constexpr int LOGE = __builtin_ctz(E);
  extern __shared__ u64 sm[];  // [N1][16]
  const u32 n = 1u << logn;
  const u32 n2 = n >> LOGN1;
  const u32 groups = n2 >> 4;
  const u32 r = blockIdx.x / groups;
  const u32 g = blockIdx.x - r * groups;
  const u32 c = threadIdx.x & 15, k = threadIdx.x >> 4;
  const u32 j = (g << 4) + c;
  const u32 pi = row_prime(in, r);
  const PrimeConst P = primes[pi];
  const ulonglong2* tw = itw_all + (u64)pi * n;
  const u64* src = row_ptr(in, r);
  u64 x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = src[j + (k * E + e) * n2];
  static_for<LOGN1 - 1, LOGE - 1, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = N1 >> (lm + 1);
    gs_stage<E, d>(x, [&](int gi) { return ldtw(tw, (1 << lm) + ((k * E + gi * 2 * d) >> (LOGN1 - lm))); },
                   P.q, P.two_q);
  });
#pragma unroll
  for (int e = 0; e < E; ++e) sm[(k * E + e) * 16 + c] = x[e];
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = sm[(k + R * e) * 16 + c];
  static_for<LOGE - 1, 0, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    gs_stage<E, (E >> (lm + 1))>(x, [&](int gi) { return ldtw(tw, (1 << lm) + gi); }, P.q, P.two_q);
  });
  // last stage (m = 1) with N^-1 folded in: x' = (x + y) N^-1, y' = (x - y) (w N^-1)
  const auto row = epi.bind(r, pi, P);
#pragma unroll
  for (int e = 0; e < E / 2; ++e) {
    const u64 a = x[e], bb = x[e + E / 2];
    x[e] = mul_shoup(a + bb, P.n_inv, P.n_inv_shoup, P.q);
    x[e + E / 2] = mul_shoup(a - bb + P.two_q, P.w1n, P.w1n_shoup, P.q);
  }
#pragma unroll
  for (int e = 0; e < E; ++e) row(j + (k + R * e) * n2, x[e]);
}

// ------------------------------------------------------------ fused column pass
// Inverse column pass of one source row + centred lift + forward column pass
// of each of its `fan` destination rows (ModUp digits, ModDown / rescale
// lifts). The inverse pass ends with thread (c, k) holding rows k + R e of
// its column -- exactly the layout the forward pass starts from -- so the
// coefficient-domain row never leaves registers: one kernel replaces the
// inverse column pass, its HBM round trip and the lift's fan-out re-reads.
//   src: rows after the inverse block pass (ntt_blk_inv), prime = source prime
//   dst: destination rows, dst row = src_row * fan + f, prime from dst.prime_of
template <int LOGN1, int E>
__global__ void __launch_bounds__(16 * ((1 << LOGN1) / E))
    ntt_col_inv_lift_fwd(const __grid_constant__ RowMap src, const __grid_constant__ RowMap dst,
                         u32 fan, const ulonglong2* __restrict__ tw_all,
                         const ulonglong2* __restrict__ itw_all,
                         const PrimeConst* __restrict__ primes, const u64* __restrict__ smod,
                         u32 nprimes, u32 logn) {
  constexpr int N1 = 1 << LOGN1;
  constexpr int R = N1 / E;
  constexpr int LOGE = __builtin_ctz(E);
  extern __shared__ u64 sm[];  // [N1][16]
  const u32 n = 1u << logn;
  const u32 n2 = n >> LOGN1;
  const u32 groups = n2 >> 4;
  const u32 rs = blockIdx.x / groups;
  const u32 g = blockIdx.x - rs * groups;
  const u32 c = threadIdx.x & 15, k = threadIdx.x >> 4;
  const u32 j = (g << 4) + c;
  const u32 ps = row_prime(src, rs);
  u64 v[E];  // coefficient-domain source values, rows k + R e
  {
    const PrimeConst S = primes[ps];
    const ulonglong2* itw = itw_all + (u64)ps * n;
    const u64* in = row_ptr(src, rs);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = in[j + (k * E + e) * n2];
    static_for<LOGN1 - 1, LOGE - 1, -1>([&](auto LM) {
      constexpr int lm = decltype(LM)::value;
      constexpr int d = N1 >> (lm + 1);
      gs_stage<E, d>(v, [&](int gi) { return ldtw(itw, (1 << lm) + ((k * E + gi * 2 * d) >> (LOGN1 - lm))); },
                     S.q, S.two_q);
    });
#pragma unroll
    for (int e = 0; e < E; ++e) sm[(k * E + e) * 16 + c] = v[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = sm[(k + R * e) * 16 + c];
    static_for<LOGE - 1, 0, -1>([&](auto LM) {
      constexpr int lm = decltype(LM)::value;
      gs_stage<E, (E >> (lm + 1))>(v, [&](int gi) { return ldtw(itw, (1 << lm) + gi); }, S.q, S.two_q);
    });
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const u64 a = v[e], bb = v[e + E / 2];
      v[e] = mul_shoup(a + bb, S.n_inv, S.n_inv_shoup, S.q);
      v[e + E / 2] = mul_shoup(a - bb + S.two_q, S.w1n, S.w1n_shoup, S.q);
    }
  }
  const u64 qs_half = __ldg(&primes[ps].half);
#pragma unroll 1
  for (u32 f = 0; f < fan; ++f) {
    const u32 rd = rs * fan + f;
    const u32 pd = row_prime(dst, rd);
    const PrimeConst P = primes[pd];
    const ulonglong2* tw = tw_all + (u64)pd * n;
    const u64 corr = P.q - __ldg(smod + ps * nprimes + pd);
    u64 x[E];
    // centred lift (rns.cpp:370-378) with the 32x32 Barrett of LiftLoad
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const u64 s = v[e];
      const u64 qh = ((u64)(u32)(s >> 24) * P.mu56) >> 32;
      u64 w = s - qh * P.q;
      if (s > qs_half) w += corr;
      x[e] = w;
    }
    static_for<0, LOGE, 1>([&](auto LM) {
      constexpr int lm = decltype(LM)::value;
      ct_stage<E, (E >> (lm + 1))>(x, [&](int gi) { return ldtw(tw, (1 << lm) + gi); }, P.q, P.two_q);
    });
    __syncthreads();  // the previous user of sm[] is done
#pragma unroll
    for (int e = 0; e < E; ++e) sm[(k + R * e) * 16 + c] = x[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = sm[(k * E + e) * 16 + c];
    static_for<LOGE, LOGN1, 1>([&](auto LM) {
      constexpr int lm = decltype(LM)::value;
      constexpr int d = N1 >> (lm + 1);
      ct_stage<E, d>(x, [&](int gi) { return ldtw(tw, (1 << lm) + ((k * E + gi * 2 * d) >> (LOGN1 - lm))); },
                     P.q, P.two_q);
    });
    u64* o = row_ptr(dst, rd);
#pragma unroll
    for (int e = 0; e < E; ++e) o[j + (k * E + e) * n2] = x[e];
  }
}

// Single-CTA transform for small rings (N <= 4096): the whole row in shared
// memory, reference stage order.
template <bool INV, class Loader, class Epi>
__global__ void __launch_bounds__(256)
    ntt_small(const __grid_constant__ Loader ld, const __grid_constant__ Epi epi,
              const __grid_constant__ RowMap rows, const ulonglong2* __restrict__ tw_all,
              const PrimeConst* __restrict__ primes, u32 logn) {
  extern __shared__ u64 smem[];
  const u32 n = 1u << logn;
  const u32 r = blockIdx.x;
  const u32 pi = row_prime(rows, r);
  const PrimeConst P = primes[pi];
  const ulonglong2* tw = tw_all + (u64)pi * n;
  {
    const auto row = ld.bind(r, pi, P);
    for (u32 a = threadIdx.x; a < n; a += blockDim.x) smem[a] = row(a);
  }
  __syncthreads();
  const auto out = epi.bind(r, pi, P);
  if (!INV) {
    u32 half = n;
    for (u32 m = 1; m < n; m <<= 1) {
      half >>= 1;
      for (u32 bt = threadIdx.x; bt < n / 2; bt += blockDim.x) {
        const u32 i = bt / half, jj = bt - i * half;
        const u32 a0 = 2 * i * half + jj;
        ct_bfly(smem[a0], smem[a0 + half], ldtw(tw, m + i), P.q, 2 * P.two_q);
      }
      __syncthreads();
    }
    for (u32 a = threadIdx.x; a < n; a += blockDim.x) out(a, reduce62(smem[a], P.q, P.mu62));
  } else {
    u32 half = 1;
    for (u32 m = n >> 1; m >= 1; m >>= 1) {
      for (u32 bt = threadIdx.x; bt < n / 2; bt += blockDim.x) {
        const u32 i = bt / half, jj = bt - i * half;
        const u32 a0 = 2 * i * half + jj;
        gs_bfly(smem[a0], smem[a0 + half], ldtw(tw, m + i), P.q, P.two_q);
      }
      __syncthreads();
      half <<= 1;
    }
    for (u32 a = threadIdx.x; a < n; a += blockDim.x)
      out(a, mul_shoup(smem[a], P.n_inv, P.n_inv_shoup, P.q));
  }
}

}  // namespace lcl
