// Negacyclic NTT over the RNS primes for sm_100a.
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
// N^-1 scaling into the column pass's last stage.
//
// Two arithmetic fields, chosen per row (per CTA) by the prime:
//   IntF  64-bit integer Harvey/Shoup butterflies on the IMAD pipe (any prime
//         < 2^55; the 54-bit special prime always runs here);
//   FpF   exact integer-valued doubles on the FP64 pipe (primes < 2^46: the
//         44/40-bit q-chain), see common.cuh "FP64 residue arithmetic".
// Both produce the same fully reduced words at every observable boundary.
// Between the two passes of one transform the row is stored in the field's
// own lazy representation (u64 words or double bits): producer and consumer
// of an intermediate always agree because both read NttTabs::fp_mask.
// Loader / epilogue functors fuse the ModUp lift, the ModDown / rescale
// divide-and-round and the key-switch output adds into the first / last
// pass, so no standalone elementwise kernel touches HBM.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace lcl {

__device__ __forceinline__ bool row_fp(const NttTabs& t, u32 pi) { return (t.fp_mask >> pi) & 1u; }
// Field selection of a launch (template argument FS): 0 = per row at run
// time, 1 = every row on the FP64 pipe, 2 = every row on the integer pipe.
// A launch whose rows share one field compiles only that field's code (the
// two-field kernels are 80-140 KB of SASS and stalled on instruction fetch).
template <int FS>
__device__ __forceinline__ bool use_fp(const NttTabs& t, u32 pi) {
  if constexpr (FS == 1) return true;
  else if constexpr (FS == 2) return false;
  else return row_fp(t, pi);
}

// ------------------------------------------------------------ fields
struct IntF {
  using T = u64;
  using TwPtr = const ulonglong2*;
  struct Tw {
    u64 w, ws;
  };
  struct K {
    u64 q, two_q, four_q;
    u32 mu62;
  };
  __device__ static __forceinline__ K konst(const PrimeConst& P) {
    return K{P.q, P.two_q, 2 * P.two_q, P.mu62};
  }
  __device__ static __forceinline__ TwPtr table(const NttTabs& t, bool inv, u32 pi) {
    return (inv ? t.itw : t.tw) + ((u64)pi << t.logn);
  }
  __device__ static __forceinline__ TwPtr btable(const NttTabs& t, bool inv, u32 pi) {
    return (inv ? t.bitw : t.btw) + ((u64)pi << t.logn);
  }
  __device__ static __forceinline__ Tw ld(TwPtr t, u32 idx) {
    const ulonglong2 v = __ldg(t + idx);
    return Tw{v.x, v.y};
  }
  // Forward CT butterfly without intermediate reduction: with t = y*w mod q
  // in [0, 4q) (truncated Shoup quotient), x' = x + t and y' = x + 4q - t stay
  // below B + 4q when x < B; from inputs < 3q, after 17 stages every value is
  // < 71q < 2^62 for q < 2^55, so the only reduction is the final one.
  __device__ static __forceinline__ void ct(T& x, T& y, Tw w, const K& k) {
    const u64 t = mul_shoup_lazy4(y, w.w, w.ws, k.q);
    const u64 a = x;
    x = a + t;
    y = a + (k.four_q - t);
  }
  // Inverse GS butterfly: x, y in [0, 4q) -> x', y' in [0, 4q) (the
  // truncated-quotient Shoup product lands in [0, 4q) too).
  __device__ static __forceinline__ void gs(T& x, T& y, Tw w, const K& k) {
    const u64 a = x, b = y;
    const u64 s = a + b;
    x = s >= k.four_q ? s - k.four_q : s;
    y = mul_shoup_lazy4(a + (k.four_q - b), w.w, w.ws, k.q);
  }
  template <int E>
  __device__ static __forceinline__ void gs_fix(T (&)[E], const K&) {}  // GS stays in [0, 4q)
  __device__ static __forceinline__ T from_u64(u64 v) { return v; }
  __device__ static __forceinline__ u64 bits(T v) { return v; }
  __device__ static __forceinline__ T unbits(u64 v) { return v; }
  __device__ static __forceinline__ u64 canon(T v, const K& k) { return reduce62(v, k.q, k.mu62); }
  // Last inverse stage with N^-1 folded in: fully reduced outputs (inputs
  // in [0, 4q)).
  __device__ static __forceinline__ void inv_last(T& a, T& b, const PrimeConst& P) {
    const u64 x = a, y = b;
    a = mul_shoup(x + y, P.n_inv, P.n_inv_shoup, P.q);
    b = mul_shoup(x - y + 2 * P.two_q, P.w1n, P.w1n_shoup, P.q);
  }
  __device__ static __forceinline__ u64 canon_last(T v, const K&) { return v; }
};

struct FpF {
  using T = double;
  using TwPtr = const double2*;
  struct Tw {
    double w, wq;
  };
  struct K {
    double q, qinv;
    u64 qi;
  };
  __device__ static __forceinline__ K konst(const PrimeConst& P) { return K{P.qf, P.qinvf, P.q}; }
  __device__ static __forceinline__ TwPtr table(const NttTabs& t, bool inv, u32 pi) {
    return (inv ? t.itwf : t.twf) + ((u64)pi << t.logn);
  }
  __device__ static __forceinline__ TwPtr btable(const NttTabs& t, bool inv, u32 pi) {
    return (inv ? t.bitwf : t.btwf) + ((u64)pi << t.logn);
  }
  __device__ static __forceinline__ Tw ld(TwPtr t, u32 idx) {
    const double2 v = __ldg(t + idx);
    return Tw{v.x, v.y};
  }
  // |t| <= 0.75q, so forward values grow by at most 0.75q per stage: from
  // inputs below 8q (lifts of a wider q-chain prime), 17 stages stay < 22q.
  __device__ static __forceinline__ void ct(T& x, T& y, Tw w, const K& k) {
    const double t = f_mulmod(y, w.w, w.wq, k.q);
    const double a = x;
    x = __dadd_rn(a, t);
    y = __dadd_rn(a, -t);
  }
  // Sums double per stage; gs_fix (every <= 4 stages) brings them back to
  // 0.75q, so every operand stays below 24q.
  __device__ static __forceinline__ void gs(T& x, T& y, Tw w, const K& k) {
    const double a = x, b = y;
    x = __dadd_rn(a, b);
    y = f_mulmod(__dadd_rn(a, -b), w.w, w.wq, k.q);
  }
  template <int E>
  __device__ static __forceinline__ void gs_fix(T (&x)[E], const K& k) {
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = f_reduce(x[e], k.q, k.qinv);
  }
  __device__ static __forceinline__ T from_u64(u64 v) { return u2d(v); }
  __device__ static __forceinline__ u64 bits(T v) { return (u64)__double_as_longlong(v); }
  __device__ static __forceinline__ T unbits(u64 v) { return __longlong_as_double((long long)v); }
  __device__ static __forceinline__ u64 canon(T v, const K& k) { return d_canon(v, k.q, k.qinv, k.qi); }
  __device__ static __forceinline__ void inv_last(T& a, T& b, const PrimeConst& P) {
    const double x = a, y = b;
    a = f_mulmod(__dadd_rn(x, y), P.ninvf, P.ninvq, P.qf);
    b = f_mulmod(__dadd_rn(x, -y), P.w1nf, P.w1nq, P.qf);
  }
  __device__ static __forceinline__ u64 canon_last(T v, const K& k) { return canon(v, k); }
};

// Padded shared-memory slot of block element i (bank-conflict-free for both
// the l + 16 e and the 16 l + e access patterns).
__device__ __forceinline__ u32 pad16(u32 i) { return i + (i >> 4); }

// ------------------------------------------------------------ loaders
// A loader is bound once per row (all address / constant lookups hoisted):
//   auto row = ld.bind(r, dst_prime_index, dst);  row(a) -> u64 congruent
// to the input, below 3q (below 2^52 for FP64 rows).
struct PlainLoad {
  RowMap in;
  struct Row {
    const u64* p;
    __device__ __forceinline__ u64 operator()(u32 a) const { return __ldg(p + a); }
  };
  __device__ __forceinline__ Row bind(u32 r, u32, const PrimeConst&) const {
    return Row{row_ptr(in, r)};
  }
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
// congruent to the reference's lift and lies in [0, 3 q_d).
// With SIGMA the source is read through the Galois automorphism X -> X^elt in
// the coefficient domain (entry = src index | negate << 31); lifting commutes
// with that signed permutation (small rings only; the two-pass rings apply the
// permutation block-locally in the evaluation domain).
__device__ __forceinline__ u64 int_lift(u64 v, u64 half, u64 corr, u64 q, u32 mu) {
  const u64 qh = ((u64)(u32)(v >> 24) * mu) >> 32;
  u64 x = v - qh * q;
  if (v > half) x += corr;
  return x;
}

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
      return int_lift(v, half, corr, q, mu);
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
// auto row = epi.bind(r, dst_prime_index, dst);  row(a, value)
// kNeedsReduced: the value is fully reduced in [0, q); otherwise an integer
// row may hand over its lazy word (< 80q); FP64 rows always hand over [0, q).
struct PlainStore {
  static constexpr bool kNeedsReduced = true;
  static constexpr bool kInvNext = false;
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
  static constexpr bool kInvNext = false;
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
    __device__ __forceinline__ u64 store(const Pre& p, u32 a, u64 lift) const {
      // lift < 80q (lazy NTT output): x + 80q - lift > 0 and congruent
      const u64 v = add_mod(mul_shoup(p.x + (q80 - lift), iv, ivs, q), p.add, q);
      o[a] = v;
      return v;
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

// DivRoundStore that also runs the NEXT key switch's inverse block pass on the
// c1 half of every output ciphertext (items with x = 1): the final words of a
// rotation level are already in registers, so the next level's ntt_blk_inv
// over its c1 limbs (and that HBM / L2 round trip) disappears. inv_out: the
// coefficient-bound rows [B][m][N] the next ks_switch hands to its fused
// column pass (ks_switch's preinv).
struct DivRoundInvStore : DivRoundStore {
  static constexpr bool kInvNext = true;
  RowMap inv_out;  // same row structure as out; group_stride m N, item_stride 0
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
template <class F, int E, int D, class TwF>
__device__ __forceinline__ void ct_stage(typename F::T (&x)[E], const TwF& twf, const typename F::K& k) {
#pragma unroll
  for (int g = 0; g < E / (2 * D); ++g) {
    const typename F::Tw w = twf(g);
#pragma unroll
    for (int e = 0; e < D; ++e) F::ct(x[g * 2 * D + e], x[g * 2 * D + e + D], w, k);
  }
}
template <class F, int E, int D, class TwF>
__device__ __forceinline__ void gs_stage(typename F::T (&x)[E], const TwF& twf, const typename F::K& k) {
#pragma unroll
  for (int g = 0; g < E / (2 * D); ++g) {
    const typename F::Tw w = twf(g);
#pragma unroll
    for (int e = 0; e < D; ++e) F::gs(x[g * 2 * D + e], x[g * 2 * D + e + D], w, k);
  }
}

// Column-pass stage groups. Thread (c, k) of a column CTA holds rows k + R e
// (layout A) or rows k E + e (layout B) of its column.
// Forward, layout A: stages m = 1 .. E/2.
template <class F, int LOGN1, int E>
__device__ __forceinline__ void col_fwd_phase1(typename F::T (&x)[E], typename F::TwPtr tw,
                                               const typename F::K& K) {
  constexpr int LOGE = __builtin_ctz(E);
  static_for<0, LOGE, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    ct_stage<F, E, (E >> (lm + 1))>(x, [&](int gi) { return F::ld(tw, (1 << lm) + gi); }, K);
  });
}
// Forward, layout B: stages m = E .. N1/2 (distance N1/(2m) < R <= E).
template <class F, int LOGN1, int E>
__device__ __forceinline__ void col_fwd_phase2(typename F::T (&x)[E], typename F::TwPtr tw, u32 k,
                                               const typename F::K& K) {
  constexpr int LOGE = __builtin_ctz(E);
  static_for<LOGE, LOGN1, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = (1 << LOGN1) >> (lm + 1);
    ct_stage<F, E, d>(x, [&](int gi) { return F::ld(tw, (1 << lm) + ((k * E + gi * 2 * d) >> (LOGN1 - lm))); },
                      K);
  });
}
// Inverse, layout B: GS stages m = N1/2 .. E.
template <class F, int LOGN1, int E>
__device__ __forceinline__ void col_inv_phase1(typename F::T (&x)[E], typename F::TwPtr tw, u32 k,
                                               const typename F::K& K) {
  constexpr int LOGE = __builtin_ctz(E);
  static_for<LOGN1 - 1, LOGE - 1, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = (1 << LOGN1) >> (lm + 1);
    gs_stage<F, E, d>(x, [&](int gi) { return F::ld(tw, (1 << lm) + ((k * E + gi * 2 * d) >> (LOGN1 - lm))); },
                      K);
  });
}
// Inverse, layout A: GS stages m = E/2 .. 2, then the last stage (m = 1) with
// N^-1 folded in: x' = (x + y) N^-1, y' = (x - y) (w N^-1).
template <class F, int E>
__device__ __forceinline__ void col_inv_phase2(typename F::T (&x)[E], typename F::TwPtr tw,
                                               const typename F::K& K, const PrimeConst& P) {
  constexpr int LOGE = __builtin_ctz(E);
  static_for<LOGE - 1, 0, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    gs_stage<F, E, (E >> (lm + 1))>(x, [&](int gi) { return F::ld(tw, (1 << lm) + gi); }, K);
  });
#pragma unroll
  for (int e = 0; e < E / 2; ++e) F::inv_last(x[e], x[e + E / 2], P);
}

// ------------------------------------------------------------ kernels
// Column pass, forward. CTA = 16 consecutive columns x N1 rows of one row-poly.
// Thread (c, k): column c, rows k + R e (phase 1, log2 E stages in registers),
// then rows k E + e (phase 2, log2 R stages) after one shared transpose.
// Output: the field's lazy words (bits) in out.
template <class F, int LOGN1, int E, class Loader>
__device__ __forceinline__ void col_fwd_body(const RowMap& out, const Loader& ld, const NttTabs& tb,
                                             u64* sm, u32 r, u32 j, u32 c, u32 k, u32 pi) {
  constexpr int N1 = 1 << LOGN1;
  constexpr int R = N1 / E;
  const u32 n2 = (1u << tb.logn) >> LOGN1;
  const PrimeConst P = tb.primes[pi];
  const typename F::K K = F::konst(P);
  const typename F::TwPtr tw = F::table(tb, false, pi);
  typename F::T x[E];
  {
    const auto row = ld.bind(r, pi, P);
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = F::from_u64(row(j + (k + R * e) * n2));
  }
  col_fwd_phase1<F, LOGN1, E>(x, tw, K);
#pragma unroll
  for (int e = 0; e < E; ++e) sm[(k + R * e) * 16 + c] = F::bits(x[e]);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = F::unbits(sm[(k * E + e) * 16 + c]);
  col_fwd_phase2<F, LOGN1, E>(x, tw, k, K);
  u64* o = row_ptr(out, r);
#pragma unroll
  for (int e = 0; e < E; ++e) o[j + (k * E + e) * n2] = F::bits(x[e]);
}

template <int LOGN1, int E, class Loader>
__global__ void __launch_bounds__(16 * ((1 << LOGN1) / E))
    ntt_col_fwd(const __grid_constant__ RowMap out, const __grid_constant__ Loader ld,
                const __grid_constant__ NttTabs tb) {
  extern __shared__ u64 sm[];  // [N1][16]
  const u32 groups = ((1u << tb.logn) >> LOGN1) >> 4;
  const u32 r = blockIdx.x / groups;
  const u32 g = blockIdx.x - r * groups;
  const u32 c = threadIdx.x & 15, k = threadIdx.x >> 4;
  const u32 j = (g << 4) + c;
  const u32 pi = row_prime(out, r);
  if (row_fp(tb, pi))
    col_fwd_body<FpF, LOGN1, E>(out, ld, tb, sm, r, j, c, k, pi);
  else
    col_fwd_body<IntF, LOGN1, E>(out, ld, tb, sm, r, j, c, k, pi);
}

// Block-pass twiddles. Block b's 8 local stages use root[(N1 + b) 2^lm + i],
// i < 2^lm, lm = 0..7 (255 entries). In the first 4 stages (lane l holds
// elements l + 16 e) i = g is the same for all 16 lanes; in the last 4 (lane l
// holds 16 l + e) lane l needs i = l 2^(lm-4) + g, g < 2^(lm-4), so in the
// reference's order the 16 lanes would read entries 2^(lm-4) apart -- up to a
// 16-way shared-memory bank conflict (16 distinct L1 lines from global) at
// lm = 7. The context therefore keeps a block-ordered copy of the table
// (NttTabs::btw..): per block 256 entries, entry (lm, g) of lane l at
//   lm < 4:  2^lm - 1 + g                          (uniform: broadcast)
//   lm >= 4: 15 + (2^(lm-4) - 1 + g) * 16 + l      (16 consecutive entries)
// so every stage reads one contiguous 256-byte run per 16 lanes.
__host__ __device__ __forceinline__ u32 blk_tw_pos(int lm, u32 g, u32 l) {
  return lm < 4 ? (1u << lm) - 1 + g : 15 + ((1u << (lm - 4)) - 1 + g) * 16 + l;
}
constexpr int kBlkTw = 256;  // entries per block (255 used)
// The CTA's block table (4 KB, contiguous) staged into shared memory once.
template <class F>
__device__ __forceinline__ void stage_blk_tw(ulonglong2* stw, typename F::TwPtr btab_block, u32 tid,
                                             u32 nthr) {
  const ulonglong2* t = reinterpret_cast<const ulonglong2*>(btab_block);
  for (u32 k = tid; k < (u32)kBlkTw; k += nthr) stw[k] = __ldg(t + k);
}
template <class F>
struct GlobalTw {  // the block's 256 block-ordered entries straight from the table (L1 / L2)
  typename F::TwPtr tw;
  __device__ __forceinline__ typename F::Tw operator()(int lm, u32 g, u32 l) const {
    return F::ld(tw, blk_tw_pos(lm, g, l));
  }
};
template <class F>
struct SmemTw {
  const ulonglong2* stw;
  __device__ __forceinline__ typename F::Tw operator()(int lm, u32 g, u32 l) const {
    const ulonglong2 v = stw[blk_tw_pos(lm, g, l)];
    typename F::Tw w;
    if constexpr (std::is_same<F, FpF>::value) {
      w.w = __longlong_as_double((long long)v.x);
      w.wq = __longlong_as_double((long long)v.y);
    } else {
      w.w = v.x;
      w.ws = v.y;
    }
    return w;
  }
};

// Block pass body, forward: x[e] holds element l + 16 e of one 256-point
// block (coalesced order) on entry; on exit o[e] = fin(output element
// l + 16 e). Phase 1 runs local stages m' = 1..8 on s = l + 16 e, phase 2
// m' = 16..128 on s = 16 l + e after a warp-local shared transpose.
template <class F, class TwA, class Fin>
__device__ __forceinline__ void blk_fwd_body(typename F::T (&x)[16], u64 (&o)[16], u64* s,
                                             const TwA& twa, u32 l, const typename F::K& K,
                                             const Fin& fin) {
  static_for<0, 4, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    ct_stage<F, 16, (16 >> (lm + 1))>(x, [&](int gi) { return twa(lm, (u32)gi, l); }, K);
  });
#pragma unroll
  for (int e = 0; e < 16; ++e) s[l + 16 * e + e] = F::bits(x[e]);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = F::unbits(s[16 * l + e + l]);
  static_for<4, 8, 1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = 256 >> (lm + 1);
    ct_stage<F, 16, d>(x, [&](int gi) { return twa(lm, (u32)gi, l); }, K);
  });
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) s[16 * l + e + l] = fin(x[e]);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) o[e] = s[l + 16 * e + e];
  __syncwarp();
}

// Block pass body, inverse: x[e] = element l + 16 e of block b (coalesced
// order) in and out; GS stages m' = 128 .. 1 (global m = N/2 .. N1). FP64
// rows are brought back to |x| <= 0.75q after each 4-stage phase.
template <class F, class TwA>
__device__ __forceinline__ void blk_inv_body(typename F::T (&x)[16], u64* s, const TwA& twa, u32 l,
                                             const typename F::K& K) {
#pragma unroll
  for (int e = 0; e < 16; ++e) s[l + 16 * e + e] = F::bits(x[e]);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = F::unbits(s[16 * l + e + l]);
  static_for<7, 3, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    constexpr int d = 256 >> (lm + 1);
    gs_stage<F, 16, d>(x, [&](int gi) { return twa(lm, (u32)gi, l); }, K);
  });
  F::gs_fix(x, K);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) s[16 * l + e + l] = F::bits(x[e]);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = F::unbits(s[l + 16 * e + e]);
  __syncwarp();
  static_for<3, -1, -1>([&](auto LM) {
    constexpr int lm = decltype(LM)::value;
    gs_stage<F, 16, (16 >> (lm + 1))>(x, [&](int gi) { return twa(lm, (u32)gi, l); }, K);
  });
  F::gs_fix(x, K);
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
// thread, 4 blocks (of one row) per CTA. The epilogue's operands are
// prefetched before the butterflies so their latency overlaps the arithmetic.
template <class F, int LOGN1, class Epi>
__device__ __forceinline__ void blk_fwd_kernel_body(const RowMap& in, const Epi& epi, const NttTabs& tb,
                                                    u64* s, u32 r, u32 b, u32 l, u32 pi) {
  const PrimeConst P = tb.primes[pi];
  const typename F::K K = F::konst(P);
  const u64* src = row_ptr(in, r) + (b << 8);
  typename F::T x[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = F::unbits(src[l + 16 * e]);
  u64 o[16];
  const GlobalTw<F> twa{F::btable(tb, false, pi) + b * kBlkTw};
  blk_fwd_body<F>(x, o, s, twa, l, K, [&](typename F::T v) -> u64 {
    if (std::is_same<F, FpF>::value || Epi::kNeedsReduced) return F::canon(v, K);
    return F::bits(v);
  });
  const auto row = epi.bind(r, pi, P);
  row.stage(s, b, l);
  // operands of 4 elements in flight at a time: latency overlap without the
  // register cost of prefetching all 16
#pragma unroll
  for (int e0 = 0; e0 < 16; e0 += 4) {
    typename Epi::Pre pre[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) row.prefetch(pre[e], (b << 8) + l + 16 * (e0 + e), s);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (Epi::kInvNext)
        o[e0 + e] = row.store(pre[e], (b << 8) + l + 16 * (e0 + e), o[e0 + e]);
      else
        row.store(pre[e], (b << 8) + l + 16 * (e0 + e), o[e0 + e]);
    }
  }
  if constexpr (Epi::kInvNext) {
    const RowMap& om = epi.out;
    if (((r / om.rows_per_item) % om.items_per_group) == 1) {
      __syncwarp();  // s[] (permuted add2 staging) is reused by the inverse body
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = F::from_u64(o[e]);
      blk_inv_body<F>(x, s, GlobalTw<F>{F::btable(tb, true, pi) + b * kBlkTw}, l, K);
      u64* dst = row_ptr(epi.inv_out, r) + (b << 8);
#pragma unroll
      for (int e = 0; e < 16; ++e) dst[l + 16 * e] = F::bits(x[e]);
    }
  }
}

// Block pass, forward: 256-point blocks, 16 threads per block, 16 elements per
// thread, 4 consecutive blocks of one row per CTA. (4 same-prime rows per CTA
// sharing block b's twiddles through L1 was measured slower at cfg3, also
// with the conflict-free block-ordered table: ntt_blk_fwd<divround+inv>
// 7.99 -> 12.18 ms, <divround> 4.58 -> 5.38, ntt_blk_inv 3.99 -> 4.05; most
// of that was the 16-lane __syncwarp mask the divergent groups needed:
// with the full-warp barrier kept, <divround+inv> alone costs 7.99 vs 11.86 ms
// with the half-warp mask.)
template <int LOGN1, class Epi, int MINB = 1, int FS = 0>
__global__ void __launch_bounds__(64, MINB)
    ntt_blk_fwd(const __grid_constant__ RowMap in, const __grid_constant__ Epi epi,
                const __grid_constant__ NttTabs tb) {
  constexpr int N1 = 1 << LOGN1;
  __shared__ u64 sm[4][256 + 16];
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  const u32 blk_global = blockIdx.x * 4 + bw;
  const u32 r = blk_global / N1;
  const u32 b = blk_global - r * N1;
  const u32 pi = row_prime(in, r);
  if (use_fp<FS>(tb, pi))
    blk_fwd_kernel_body<FpF, LOGN1>(in, epi, tb, sm[bw], r, b, l, pi);
  else
    blk_fwd_kernel_body<IntF, LOGN1>(in, epi, tb, sm[bw], r, b, l, pi);
}

// Divide-and-round block pass with its operands staged by TMA. The 16-lane
// group of block b issues, from one lane, cp.async.bulk copies of every
// 2 KB block it needs -- the ModDown column-pass output (mid), the key-switch
// accumulator x, add1 and add2's (Galois-)source block -- onto one mbarrier
// before it does anything else, so the epilogue's loads are in flight during
// the block stages instead of being issued (and waited for) after them.
// Shared memory per group: [272] mid (later the transpose buffer), [256] x,
// [256] add1, [256] add2, mbarrier.
constexpr int kDrGroupWords = 272 + 3 * 256 + 2;
template <class F, int LOGN1, class Epi>
__device__ __forceinline__ void blk_fwd_dr_tma_body(const RowMap& in, const Epi& epi, const NttTabs& tb,
                                                    u64* g, u32 r, u32 b, u32 l, u32 pi) {
  const PrimeConst P = tb.primes[pi];
  const typename F::K K = F::konst(P);
  const auto row = epi.bind(r, pi, P);
  u64* smid = g;
  u64* sx = g + 272;
  u64* sa1 = sx + 256;
  u64* sa2 = sa1 + 256;
  u64* bar = sa2 + 256;
  const u32 bo = b << 8;
  if (l == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, 2048u * (2 + (row.a1 ? 1 : 0) + (row.a2 ? 1 : 0)));
    bulk_g2s(smid, row_ptr(in, r) + bo, 2048, bar);
    bulk_g2s(sx, row.x + bo, 2048, bar);
    if (row.a1) bulk_g2s(sa1, row.a1 + bo, 2048, bar);
    if (row.a2) bulk_g2s(sa2, row.a2 + (row.perm ? (__ldg(row.perm + bo) & ~255u) : bo), 2048, bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  typename F::T x[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = F::unbits(smid[l + 16 * e]);
  __syncwarp();  // smid becomes the transpose buffer
  u64 o[16];
  const GlobalTw<F> twa{F::btable(tb, false, pi) + b * kBlkTw};
  blk_fwd_body<F>(x, o, smid, twa, l, K, [&](typename F::T v) -> u64 {
    if (std::is_same<F, FpF>::value || Epi::kNeedsReduced) return F::canon(v, K);
    return F::bits(v);
  });
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const u32 a = l + 16 * e;
    u64 add = row.a1 ? sa1[a] : 0;
    if (row.a2) add = add_mod(add, sa2[row.perm ? (__ldg(row.perm + bo + a) & 255u) : a], row.q);
    const u64 v = add_mod(mul_shoup(sx[a] + (row.q80 - o[e]), row.iv, row.ivs, row.q), add, row.q);
    row.o[bo + a] = v;
    o[e] = v;
  }
  if constexpr (Epi::kInvNext) {
    const RowMap& om = epi.out;
    if (((r / om.rows_per_item) % om.items_per_group) == 1) {
      __syncwarp();
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = F::from_u64(o[e]);
      blk_inv_body<F>(x, smid, GlobalTw<F>{F::btable(tb, true, pi) + b * kBlkTw}, l, K);
      u64* dst = row_ptr(epi.inv_out, r) + bo;
#pragma unroll
      for (int e = 0; e < 16; ++e) dst[l + 16 * e] = F::bits(x[e]);
    }
  }
}

template <int LOGN1, class Epi, int MINB>
__global__ void __launch_bounds__(64, MINB)
    ntt_blk_fwd_dr_tma(const __grid_constant__ RowMap in, const __grid_constant__ Epi epi,
                       const __grid_constant__ NttTabs tb) {
  constexpr int N1 = 1 << LOGN1;
  extern __shared__ __align__(16) u64 dr_sm[];  // [4][kDrGroupWords]
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  const u32 blk_global = blockIdx.x * 4 + bw;
  const u32 r = blk_global / N1;
  const u32 b = blk_global - r * N1;
  const u32 pi = row_prime(in, r);
  u64* g = dr_sm + bw * kDrGroupWords;
  if (row_fp(tb, pi))
    blk_fwd_dr_tma_body<FpF, LOGN1>(in, epi, tb, g, r, b, l, pi);
  else
    blk_fwd_dr_tma_body<IntF, LOGN1>(in, epi, tb, g, r, b, l, pi);
}

// ModUp block pass fused with the key inner product (ckks.cpp:464-518).
// A 16-thread group owns block blk of target row t of ciphertext b and walks
// the M digits: digit j is the column-pass output mid[b][j][t'] run through
// the block stages, except the identity row t == j, whose lifted NTT is the
// input limb itself (mod_up returns the row unchanged, rns.cpp:371-381), read
// through the rotation's evaluation-domain permutation when one is given.
// Each digit is multiplied by the key and accumulated lazily, so the m(m+1)
// digit rows never reach HBM. Integer rows use the key in Shoup form
// (key_aux = floor(k 2^64 / q)); FP64 rows read only key_aux = the key word
// as a double (one load per key word).
//   mid: [B][M][M][N] (t' = t < j ? t : t - 1); c1: limb j of item b at
//   c1 + b * c1_stride + j * N; key / key_aux: [full][2][full+1][N];
//   acc: [B][2][M+1][N].
template <class F>
struct IpOps;
template <>
struct IpOps<IntF> {
  static constexpr bool kRawKey = true;
  // each product < 4q: the M-term sums stay < 24q (M <= 6)
  __device__ static __forceinline__ u64 mul(u64 x, u64 k, u64 ks, const IntF::K& K) {
    return mul_shoup_lazy4(x, k, ks, K.q);
  }
  __device__ static __forceinline__ u64 add(u64 a, u64 b) { return a + b; }
};
template <>
struct IpOps<FpF> {
  // kd = the key word as a double; w / q is formed as kd * fl(1 / q), within
  // 2^-52 relative of k / q, so for |x| < 2^49 (lazy forward outputs < 22q)
  // round(x * wq) stays within 0.625 of x k / q -- f_mulmod's 0.75 bound --
  // and each product is exact with |p| <= 0.75q. The raw key word is unused.
  static constexpr bool kRawKey = false;
  __device__ static __forceinline__ u64 mul(double x, u64, u64 kd_bits, const FpF::K& K) {
    const double kd = __longlong_as_double((long long)kd_bits);
    return (u64)__double_as_longlong(f_mulmod(x, kd, __dmul_rn(kd, K.qinv), K.q));
  }
  __device__ static __forceinline__ u64 add(u64 a, u64 b) {
    return (u64)__double_as_longlong(__dadd_rn(__longlong_as_double((long long)a),
                                               __longlong_as_double((long long)b)));
  }
};

// LCL_MODUP_KEYS selects how the key words reach the inner product:
//   0  __ldg per element (L1 serves the CTA's 4 groups);
//   1  as 0, plus cp.async.bulk.prefetch.L2 of digit j+1's key rows and mid
//      block while digit j transforms;
//   2  TMA: the (target row, block) key rows of digit j are bulk-copied into
//      shared memory (cp.async.bulk + mbarrier) by one thread, overlapping
//      digit j's block stages; the buffer is refilled for j+1 after a CTA
//      barrier.
// Measured at cfg3 (modup_ip_blk<perm>, 13 levels x 190 ciphertexts): 0
// 12.77 ms, 1 12.80, 2 13.31 -- the key words are L2 hits shared by the
// CTA's 4 groups, and the 8 KB staging buffer costs one CTA per SM (6 vs 7),
// so 0 is the default; 1 and 2 stay parity-tested (tools/build_variant.sh).
#ifndef LCL_MODUP_KEYS
#define LCL_MODUP_KEYS 0
#endif
// (Measured and rejected at cfg3, modup_ip_blk<perm>, 13 levels: a register
// software pipeline loading digit j + 1's block while digit j computes,
// 12.84 -> 13.47 ms at 6 CTAs/SM and 14.62 at 8; 2 or 4 ciphertext quads per
// CTA so the staged twiddles are reused, 12.93 / 12.95 ms; after the
// block-ordered twiddles (11.48 ms), the accumulators in registers instead
// of shared memory, 13.09 ms at 6 CTAs/SM and 14.80 at 8.)

template <class F, int LOGN1, int M>
__device__ __forceinline__ void modup_ip_body(u32 bi, bool live, u32 t, u32 blk, u32 pi, u32 l,
                                              u64* s, u64* s0acc, u64* s1acc, ulonglong2* stw,
                                              const u64* mid,
                                              const u64* c1, u64 c1_stride, const u32* perm,
                                              const u64* key, const u64* key_aux, u32 full,
                                              u64* acc, const NttTabs& tb, u64 (*skey)[256],
                                              u64* kbar) {
  const u32 n = 1u << tb.logn;
  const PrimeConst P = tb.primes[pi];
  const typename F::K K = F::konst(P);
  const u64 kstride = (u64)(full + 1) * n;
  const u32 a0 = (blk << 8) + l;
  // rotation: output block blk of every digit comes from block src_blk of the
  // unpermuted digit (block-local Galois permutation, see block_gather)
  const u32 src_blk = perm ? (__ldg(perm + (blk << 8)) >> 8) : blk;
  constexpr u32 kRows = IpOps<F>::kRawKey ? 4 : 2;  // key rows the field reads per digit
  auto key_rows = [&](int j, u32 r) -> const u64* {
    const u64 off = (2ull * j + (r & 1)) * kstride + (u64)pi * n + (blk << 8);
    return (IpOps<F>::kRawKey && r < 2 ? key : key_aux) + off;
  };
  if constexpr (LCL_MODUP_KEYS == 2) {
    if (threadIdx.x == 0) {
      mbar_init(kbar, 1);
      mbar_expect_tx(kbar, kRows * 2048);
      for (u32 r = 0; r < kRows; ++r) bulk_g2s(skey[r], key_rows(0, r), 2048, kbar);
    }
  }
  // the CTA's 4 groups share (target row, block): its twiddles are staged once
  stage_blk_tw<F>(stw, F::btable(tb, false, pi) + src_blk * kBlkTw, threadIdx.x, blockDim.x);
  __syncthreads();
  const SmemTw<F> twa{stw};
#pragma unroll 1
  for (int j = 0; j < M; ++j) {
    if constexpr (LCL_MODUP_KEYS == 1) {
      if (j + 1 < M) {
        if (threadIdx.x < kRows) bulk_prefetch_l2(key_rows(j + 1, threadIdx.x), 2048);
        if (l == 0 && t != (u32)(j + 1)) {
          const u32 tp = t < (u32)(j + 1) ? t : t - 1;
          bulk_prefetch_l2(mid + (((u64)bi * M + j + 1) * M + tp) * n + (src_blk << 8), 2048);
        }
      }
    }
    typename F::T x[16];
    if (t == (u32)j) {
      const u64* src = c1 + (u64)bi * c1_stride + (u64)j * n + (src_blk << 8);
      u64 v[16];
      if (perm) {
        block_gather(v, s, src, perm, blk, l);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = __ldg(src + l + 16 * e);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = F::from_u64(v[e]);
    } else {
      const u32 tp = t < (u32)j ? t : t - 1;
      const u64* src = mid + (((u64)bi * M + j) * M + tp) * n + (src_blk << 8);
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = F::unbits(src[l + 16 * e]);
      u64 o[16];
      blk_fwd_body<F>(x, o, s, twa, l, K, [](typename F::T v) { return F::bits(v); });
      if (perm) {
        // the body left the (lazy) block in shared memory: permuted read
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = F::unbits(s[pad16(__ldg(perm + (blk << 8) + l + 16 * e) & 255u)]);
        __syncwarp();
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = F::unbits(o[e]);
      }
    }
    if constexpr (LCL_MODUP_KEYS == 2) {
      mbar_wait(kbar, (u32)j & 1u);
      constexpr u32 A = IpOps<F>::kRawKey ? 2 : 0;  // shared rows of the Shoup / double words
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const u32 si = l + 16 * e;
        const u64 kw0 = IpOps<F>::kRawKey ? skey[0][si] : 0;
        const u64 kw1 = IpOps<F>::kRawKey ? skey[1][si] : 0;
        const u64 p0 = IpOps<F>::mul(x[e], kw0, skey[A][si], K);
        const u64 p1 = IpOps<F>::mul(x[e], kw1, skey[A + 1][si], K);
        s0acc[si] = j ? IpOps<F>::add(s0acc[si], p0) : p0;
        s1acc[si] = j ? IpOps<F>::add(s1acc[si], p1) : p1;
      }
      __syncthreads();  // every group has read digit j's keys
      if (j + 1 < M && threadIdx.x == 0) {
        fence_proxy_async();
        mbar_expect_tx(kbar, kRows * 2048);
        for (u32 r = 0; r < kRows; ++r) bulk_g2s(skey[r], key_rows(j + 1, r), 2048, kbar);
      }
    } else {
      const u64* k0 = key + (2ull * j) * kstride + (u64)pi * n;
      const u64* k1 = k0 + kstride;
      const u64* ks0 = key_aux + (2ull * j) * kstride + (u64)pi * n;
      const u64* ks1 = ks0 + kstride;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const u32 a = a0 + 16 * e;
        const u64 kw0 = IpOps<F>::kRawKey ? __ldg(k0 + a) : 0;
        const u64 kw1 = IpOps<F>::kRawKey ? __ldg(k1 + a) : 0;
        const u64 p0 = IpOps<F>::mul(x[e], kw0, __ldg(ks0 + a), K);
        const u64 p1 = IpOps<F>::mul(x[e], kw1, __ldg(ks1 + a), K);
        const u32 si = l + 16 * e;
        s0acc[si] = j ? IpOps<F>::add(s0acc[si], p0) : p0;
        s1acc[si] = j ? IpOps<F>::add(s1acc[si], p1) : p1;
      }
    }
  }
  if (!live) return;
  u64* o0 = acc + ((u64)bi * 2 * (M + 1) + t) * n;
  u64* o1 = o0 + (u64)(M + 1) * n;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const u32 si = l + 16 * e;
    o0[a0 + 16 * e] = F::canon(F::unbits(s0acc[si]), K);
    o1[a0 + 16 * e] = F::canon(F::unbits(s1acc[si]), K);
  }
}

// LCL_MODUP_G: 16-lane groups (ciphertexts) per CTA; MINB keeps 128
// registers. 8 groups (4 CTAs / SM, 16 warps, 53 KB shared) against 4 (7
// CTAs / SM: shared-memory bound, 14 warps): cfg3 modup_ip_blk<perm>
// 11.28 -> 10.53 ms, relinearisation 3.44 -> 3.29 ms.
#ifndef LCL_MODUP_G
#define LCL_MODUP_G 8
#endif
constexpr size_t modup_smem_bytes(int G) { return (size_t)G * (256 + 16 + 512) * 8 + kBlkTw * 16; }
// FS (see use_fp): 0 = all M + 1 targets in one launch (t0 = 0), 2 = the
// special target only, 1 = the M q targets only (t0 = 1): the field-split
// launches compile one field each.
template <int LOGN1, int M, int FS = 0, int G = LCL_MODUP_G, int MINB = 32 / G>
__global__ void __launch_bounds__(16 * G, MINB)
    modup_ip_blk(u32 B, const u64* __restrict__ mid, const u64* __restrict__ c1, u64 c1_stride,
                 const u32* __restrict__ perm, const u64* __restrict__ key,
                 const u64* __restrict__ key_aux, u32 full, u64* __restrict__ acc,
                 const __grid_constant__ NttTabs tb, u32 t0) {
  constexpr int N1 = 1 << LOGN1;
  // dynamic shared memory (modup_smem_bytes): [G][272] block transposes,
  // [G][2][256] lazy accumulators (coalesced order), the block's twiddles
  extern __shared__ u64 dyn_sm[];
  u64(*sm)[256 + 16] = reinterpret_cast<u64(*)[256 + 16]>(dyn_sm);
  u64(*sacc)[2][256] = reinterpret_cast<u64(*)[2][256]>(dyn_sm + G * (256 + 16));
  ulonglong2* stw = reinterpret_cast<ulonglong2*>(dyn_sm + G * (256 + 16 + 512));
#if LCL_MODUP_KEYS == 2
  __shared__ alignas(128) u64 skey[4][256];  // digit j's key rows (TMA)
  __shared__ u64 kbar;
#else
  u64(*skey)[256] = nullptr;
  u64* kbar_p = nullptr;
#endif
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  // the G groups of a CTA take G consecutive ciphertexts of the same
  // (target row, block): the key words they share are served from L1 and
  // the block's twiddles are staged once
  const u32 bq_count = (B + G - 1) / G;
  const u32 bq = blockIdx.x % bq_count;
  const u32 tb_ = blockIdx.x / bq_count;  // = t * N1 + blk
  // the special-prime target (integer field, the slowest CTAs) is scheduled
  // first so its CTAs overlap the q targets instead of forming the tail
  const u32 tr = tb_ / N1, blk = tb_ - tr * N1;
  const u32 traw = tr + t0;
  const u32 t = traw == 0 ? (u32)M : traw - 1;
  const u32 pi = t < (u32)M ? t : full;
#if LCL_MODUP_KEYS == 2
  u64* kbar_p = &kbar;
#endif
  // groups past the batch redo item B - 1 without storing (the block stages
  // use warp-wide barriers)
  const u32 bi_raw = bq * G + bw;
  const bool live = bi_raw < B;
  const u32 bi = live ? bi_raw : B - 1;
  if (use_fp<FS>(tb, pi))
    modup_ip_body<FpF, LOGN1, M>(bi, live, t, blk, pi, l, sm[bw], sacc[bw][0], sacc[bw][1], stw, mid, c1,
                                 c1_stride, perm, key, key_aux, full, acc, tb, skey, kbar_p);
  else
    modup_ip_body<IntF, LOGN1, M>(bi, live, t, blk, pi, l, sm[bw], sacc[bw][0], sacc[bw][1], stw, mid, c1,
                                  c1_stride, perm, key, key_aux, full, acc, tb, skey, kbar_p);
}

// Hoisted rotations (ckks.cpp:582-612) fused like modup_ip_blk: ONE ModUp
// block pass feeds the inner products of up to kHoistMax rotation steps.
// A 16-thread group owns SOURCE block sb of target row t of item b: it runs
// the block stages of the M digits once (the identity digit t == j is the
// input limb's block, unpermuted) and keeps them in shared memory; then for
// every step s the Galois permutation maps source block sb onto exactly one
// output block ob = blkmap_s[sb] (block-local, see block_gather), whose
// elements are gathered from the staged digits, multiplied by the step's
// key words and accumulated over the digits in registers. The m(m+1) digit
// rows never reach HBM and are transformed once for all the steps.
//   mid: [B][M][M][N] (as modup_ip_blk); acc: step s at acc + s * acc_step,
//   [B][2][M+1][N] each.
constexpr int kHoistMax = 8;
struct HoistSteps {
  const u32* perm[kHoistMax];
  const u32* blkmap[kHoistMax];
  const u64* key[kHoistMax];
  const u64* key_aux[kHoistMax];
};

template <class F, int LOGN1, int M>
__device__ __forceinline__ void modup_ip_hoist_body(u32 bi, bool live, u32 t, u32 sb, u32 pi,
                                                    u32 l, u64* s, u64 (*sd)[256 + 16],
                                                    ulonglong2* stw, const u64* mid,
                                                    const u64* c1, u64 c1_stride,
                                                    const HoistSteps& hs, u32 nsteps, u32 full,
                                                    u64* acc, u64 acc_step, const NttTabs& tb) {
  const u32 n = 1u << tb.logn;
  const PrimeConst P = tb.primes[pi];
  const typename F::K K = F::konst(P);
  const u64 kstride = (u64)(full + 1) * n;
  stage_blk_tw<F>(stw, F::btable(tb, false, pi) + sb * kBlkTw, threadIdx.x, 64);
  __syncthreads();
  const SmemTw<F> twa{stw};
#pragma unroll 1
  for (int j = 0; j < M; ++j) {
    if (t == (u32)j) {
      const u64* src = c1 + (u64)bi * c1_stride + (u64)j * n + (sb << 8);
#pragma unroll
      for (int e = 0; e < 16; ++e) sd[j][pad16(l + 16 * e)] = F::bits(F::from_u64(__ldg(src + l + 16 * e)));
    } else {
      const u32 tp = t < (u32)j ? t : t - 1;
      const u64* src = mid + (((u64)bi * M + j) * M + tp) * n + (sb << 8);
      typename F::T x[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = F::unbits(src[l + 16 * e]);
      u64 o[16];
      blk_fwd_body<F>(x, o, s, twa, l, K, [](typename F::T v) { return F::bits(v); });
#pragma unroll
      for (int e = 0; e < 16; ++e) sd[j][pad16(l + 16 * e)] = o[e];
    }
  }
  __syncwarp();
  if (!live) return;
#pragma unroll 1
  for (u32 st = 0; st < nsteps; ++st) {
    const u32 ob = __ldg(hs.blkmap[st] + sb);
    const u32* perm = hs.perm[st];
    const u64* k0 = hs.key[st] + (u64)pi * n;
    const u64* ks0 = hs.key_aux[st] + (u64)pi * n;
    u64* o0 = acc + st * acc_step + ((u64)bi * 2 * (M + 1) + t) * n;
    u64* o1 = o0 + (u64)(M + 1) * n;
#pragma unroll 4
    for (int e = 0; e < 16; ++e) {
      const u32 a = (ob << 8) + l + 16 * e;
      const u32 si = pad16(__ldg(perm + a) & 255u);
      u64 a0 = 0, a1 = 0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const u64 off = (2ull * j) * kstride + a;
        const typename F::T x = F::unbits(sd[j][si]);
        const u64 kw0 = IpOps<F>::kRawKey ? __ldg(k0 + off) : 0;
        const u64 kw1 = IpOps<F>::kRawKey ? __ldg(k0 + off + kstride) : 0;
        const u64 p0 = IpOps<F>::mul(x, kw0, __ldg(ks0 + off), K);
        const u64 p1 = IpOps<F>::mul(x, kw1, __ldg(ks0 + off + kstride), K);
        a0 = j ? IpOps<F>::add(a0, p0) : p0;
        a1 = j ? IpOps<F>::add(a1, p1) : p1;
      }
      o0[a] = F::canon(F::unbits(a0), K);
      o1[a] = F::canon(F::unbits(a1), K);
    }
  }
}

template <int LOGN1, int M, int MINB = 6>
__global__ void __launch_bounds__(64, MINB)
    modup_ip_hoist(u32 B, const u64* __restrict__ mid, const u64* __restrict__ c1, u64 c1_stride,
                   const __grid_constant__ HoistSteps hs, u32 nsteps, u32 full,
                   u64* __restrict__ acc, u64 acc_step, const __grid_constant__ NttTabs tb) {
  constexpr int N1 = 1 << LOGN1;
  __shared__ u64 sm[4][256 + 16];
  __shared__ u64 sd[4][M][256 + 16];  // the group's M transformed digit blocks
  __shared__ ulonglong2 stw[kBlkTw];
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  const u32 bq_count = (B + 3) >> 2;
  const u32 bq = blockIdx.x % bq_count;
  const u32 tb_ = blockIdx.x / bq_count;
  const u32 traw = tb_ / N1, sb = tb_ - traw * N1;
  const u32 t = traw == 0 ? (u32)M : traw - 1;  // special-prime target first
  const u32 bi_raw = bq * 4 + bw;
  const bool live = bi_raw < B;
  const u32 bi = live ? bi_raw : B - 1;
  const u32 pi = t < (u32)M ? t : full;
  if (row_fp(tb, pi))
    modup_ip_hoist_body<FpF, LOGN1, M>(bi, live, t, sb, pi, l, sm[bw], sd[bw], stw, mid, c1,
                                       c1_stride, hs, nsteps, full, acc, acc_step, tb);
  else
    modup_ip_hoist_body<IntF, LOGN1, M>(bi, live, t, sb, pi, l, sm[bw], sd[bw], stw, mid, c1,
                                        c1_stride, hs, nsteps, full, acc, acc_step, tb);
}

// Block pass, inverse: GS stages m = N/2 .. N1 (local m' = 128 .. 1). Input:
// fully reduced words; output: the field's lazy words for the column pass.
template <class F, int LOGN1>
__device__ __forceinline__ void blk_inv_kernel_body(const RowMap& in, const RowMap& out,
                                                    const NttTabs& tb, u64* s, u32 r, u32 b, u32 l,
                                                    u32 pi) {
  const typename F::K K = F::konst(tb.primes[pi]);
  const u64* src = row_ptr(in, r) + (b << 8);
  typename F::T x[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = F::from_u64(src[l + 16 * e]);
  blk_inv_body<F>(x, s, GlobalTw<F>{F::btable(tb, true, pi) + b * kBlkTw}, l, K);
  u64* dst = row_ptr(out, r) + (b << 8);
#pragma unroll
  for (int e = 0; e < 16; ++e) dst[l + 16 * e] = F::bits(x[e]);
}

template <int LOGN1, int MINB = 1, int FS = 0>
__global__ void __launch_bounds__(64, MINB)
    ntt_blk_inv(const __grid_constant__ RowMap in, const __grid_constant__ RowMap out,
                const __grid_constant__ NttTabs tb) {
  constexpr int N1 = 1 << LOGN1;
  __shared__ u64 sm[4][256 + 16];
  const u32 l = threadIdx.x & 15, bw = threadIdx.x >> 4;
  const u32 blk_global = blockIdx.x * 4 + bw;
  const u32 r = blk_global / N1;
  const u32 b = blk_global - r * N1;
  const u32 pi = row_prime(in, r);
  if (use_fp<FS>(tb, pi))
    blk_inv_kernel_body<FpF, LOGN1>(in, out, tb, sm[bw], r, b, l, pi);
  else
    blk_inv_kernel_body<IntF, LOGN1>(in, out, tb, sm[bw], r, b, l, pi);
}

// Column pass, inverse: GS stages m = N1/2 .. 1 with x N^-1 folded into the
// last one; the fully reduced result goes through the epilogue.
template <class F, int LOGN1, int E, class Epi>
__device__ __forceinline__ void col_inv_body(const RowMap& in, const Epi& epi, const NttTabs& tb,
                                             u64* sm, u32 r, u32 j, u32 c, u32 k, u32 pi) {
  constexpr int N1 = 1 << LOGN1;
  constexpr int R = N1 / E;
  const u32 n2 = (1u << tb.logn) >> LOGN1;
  const PrimeConst P = tb.primes[pi];
  const typename F::K K = F::konst(P);
  const typename F::TwPtr tw = F::table(tb, true, pi);
  const u64* src = row_ptr(in, r);
  typename F::T x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = F::unbits(src[j + (k * E + e) * n2]);
  col_inv_phase1<F, LOGN1, E>(x, tw, k, K);
  F::gs_fix(x, K);
#pragma unroll
  for (int e = 0; e < E; ++e) sm[(k * E + e) * 16 + c] = F::bits(x[e]);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = F::unbits(sm[(k + R * e) * 16 + c]);
  col_inv_phase2<F, E>(x, tw, K, P);
  const auto row = epi.bind(r, pi, P);
#pragma unroll
  for (int e = 0; e < E; ++e) row(j + (k + R * e) * n2, F::canon_last(x[e], K));
}

template <int LOGN1, int E, class Epi>
__global__ void __launch_bounds__(16 * ((1 << LOGN1) / E))
    ntt_col_inv(const __grid_constant__ RowMap in, const __grid_constant__ Epi epi,
                const __grid_constant__ NttTabs tb) {
  extern __shared__ u64 sm[];  // [N1][16]
  const u32 groups = ((1u << tb.logn) >> LOGN1) >> 4;
  const u32 r = blockIdx.x / groups;
  const u32 g = blockIdx.x - r * groups;
  const u32 c = threadIdx.x & 15, k = threadIdx.x >> 4;
  const u32 j = (g << 4) + c;
  const u32 pi = row_prime(in, r);
  if (row_fp(tb, pi))
    col_inv_body<FpF, LOGN1, E>(in, epi, tb, sm, r, j, c, k, pi);
  else
    col_inv_body<IntF, LOGN1, E>(in, epi, tb, sm, r, j, c, k, pi);
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
// The coefficient v of the source prime q_s is lifted by the reference's rule
// (centred: v > q_s / 2 means v - q_s) into each destination prime:
//   integer source: v in [0, q_s) -> int_lift (integer dest) or its double;
//   FP64 source: the exact centred double c -> c itself (FP64 dest) or
//   c mod q_d as a word (integer dest).
template <class Fs, class Fd>
__device__ __forceinline__ typename Fd::T lift_to(typename Fs::T v, u64 qs_half, u64 corr,
                                                  const PrimeConst& D) {
  if constexpr (std::is_same<Fs, IntF>::value) {
    const u64 x = int_lift(v, qs_half, corr, D.q, D.mu56);
    if constexpr (std::is_same<Fd, IntF>::value)
      return x;
    else
      return u2d(x);
  } else {
    if constexpr (std::is_same<Fd, FpF>::value) {
      return v;
    } else {
      const long long i = d2ll(v);
      return (u64)(i + ((i >> 63) & (long long)D.q));
    }
  }
}

// LCL_COL_VSMEM: the coefficient-domain source tile v is parked in a second
// shared-memory tile (thread-private slots, no barrier) across the fan-out
// instead of registers, so the register cap does not spill it to local memory.
#ifndef LCL_COL_VSMEM
#define LCL_COL_VSMEM 1
#endif
template <class Fs, class Fd, int LOGN1, int E, class VSrc>
__device__ __forceinline__ void col_lift_fwd(const VSrc& v, const RowMap& dst, u32 rd,
                                             u32 pd, u64 qs_half, u64 corr, const NttTabs& tb,
                                             u64* sm, u32 j, u32 c, u32 k) {
  constexpr int N1 = 1 << LOGN1;
  constexpr int R = N1 / E;
  const u32 n2 = (1u << tb.logn) >> LOGN1;
  const PrimeConst D = tb.primes[pd];
  const typename Fd::K K = Fd::konst(D);
  const typename Fd::TwPtr tw = Fd::table(tb, false, pd);
  typename Fd::T x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = lift_to<Fs, Fd>(v(e), qs_half, corr, D);
  col_fwd_phase1<Fd, LOGN1, E>(x, tw, K);
  __syncthreads();  // the previous user of sm[] is done
#pragma unroll
  for (int e = 0; e < E; ++e) sm[(k + R * e) * 16 + c] = Fd::bits(x[e]);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = Fd::unbits(sm[(k * E + e) * 16 + c]);
  col_fwd_phase2<Fd, LOGN1, E>(x, tw, k, K);
  u64* o = row_ptr(dst, rd);
#pragma unroll
  for (int e = 0; e < E; ++e) o[j + (k * E + e) * n2] = Fd::bits(x[e]);
}

template <class Fs, int LOGN1, int E, int FSD>
__device__ __forceinline__ void col_ilf_body(const RowMap& src, const RowMap& dst, u32 fan,
                                             const u64* smod, u32 nprimes, const NttTabs& tb,
                                             u64* sm, u32 rs, u32 j, u32 c, u32 k, u32 ps) {
  constexpr int N1 = 1 << LOGN1;
  constexpr int R = N1 / E;
  const u32 n2 = (1u << tb.logn) >> LOGN1;
  typename Fs::T v[E];  // coefficient-domain source values, rows k + R e
  {
    const PrimeConst S = tb.primes[ps];
    const typename Fs::K K = Fs::konst(S);
    const typename Fs::TwPtr itw = Fs::table(tb, true, ps);
    const u64* in = row_ptr(src, rs);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = Fs::unbits(in[j + (k * E + e) * n2]);
    col_inv_phase1<Fs, LOGN1, E>(v, itw, k, K);
    Fs::gs_fix(v, K);
#pragma unroll
    for (int e = 0; e < E; ++e) sm[(k * E + e) * 16 + c] = Fs::bits(v[e]);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = Fs::unbits(sm[(k + R * e) * 16 + c]);
    col_inv_phase2<Fs, E>(v, itw, K, S);
    if constexpr (std::is_same<Fs, FpF>::value) {
      // exact centred coefficient (|v| <= 0.75 q_s on entry)
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = f_reduce(v[e], K.q, K.qinv);
    }
  }
  const u64 qs_half = __ldg(&tb.primes[ps].half);
  u64* vs = sm + N1 * 16;  // LCL_COL_VSMEM (E = 16): thread-private slots (k + R e) * 16 + c
  if constexpr (LCL_COL_VSMEM && E == 16) {
#pragma unroll
    for (int e = 0; e < E; ++e) vs[(k + R * e) * 16 + c] = Fs::bits(v[e]);
  }
  const auto vget = [&](int e) -> typename Fs::T {
    if constexpr (LCL_COL_VSMEM && E == 16) return Fs::unbits(vs[(k + R * e) * 16 + c]);
    else return v[e];
  };
#pragma unroll 1
  for (u32 f = 0; f < fan; ++f) {
    const u32 rd = rs * fan + f;
    const u32 pd = row_prime(dst, rd);
    const u64 corr = __ldg(&tb.primes[pd].q) - __ldg(smod + ps * nprimes + pd);
    if (use_fp<FSD>(tb, pd))
      col_lift_fwd<Fs, FpF, LOGN1, E>(vget, dst, rd, pd, qs_half, corr, tb, sm, j, c, k);
    else
      col_lift_fwd<Fs, IntF, LOGN1, E>(vget, dst, rd, pd, qs_half, corr, tb, sm, j, c, k);
  }
}

template <int LOGN1, int E, int MINB = 1, int FSS = 0, int FSD = 0>
__global__ void __launch_bounds__(16 * ((1 << LOGN1) / E), MINB)
    ntt_col_inv_lift_fwd(const __grid_constant__ RowMap src, const __grid_constant__ RowMap dst,
                         u32 fan, const u64* __restrict__ smod, u32 nprimes,
                         const __grid_constant__ NttTabs tb) {
  extern __shared__ u64 sm[];  // [N1][16]
  const u32 groups = ((1u << tb.logn) >> LOGN1) >> 4;
  const u32 rs = blockIdx.x / groups;
  const u32 g = blockIdx.x - rs * groups;
  const u32 c = threadIdx.x & 15, k = threadIdx.x >> 4;
  const u32 j = (g << 4) + c;
  const u32 ps = row_prime(src, rs);
  if (use_fp<FSS>(tb, ps))
    col_ilf_body<FpF, LOGN1, E, FSD>(src, dst, fan, smod, nprimes, tb, sm, rs, j, c, k, ps);
  else
    col_ilf_body<IntF, LOGN1, E, FSD>(src, dst, fan, smod, nprimes, tb, sm, rs, j, c, k, ps);
}

// Single-CTA transform for small rings (N <= 4096): the whole row in shared
// memory, reference stage order, integer field only.
template <bool INV, class Loader, class Epi>
__global__ void __launch_bounds__(256)
    ntt_small(const __grid_constant__ Loader ld, const __grid_constant__ Epi epi,
              const __grid_constant__ RowMap rows, const __grid_constant__ NttTabs tb) {
  extern __shared__ u64 smem[];
  const u32 n = 1u << tb.logn;
  const u32 r = blockIdx.x;
  const u32 pi = row_prime(rows, r);
  const PrimeConst P = tb.primes[pi];
  const IntF::K K = IntF::konst(P);
  const IntF::TwPtr tw = IntF::table(tb, INV, pi);
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
        IntF::ct(smem[a0], smem[a0 + half], IntF::ld(tw, m + i), K);
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
        IntF::gs(smem[a0], smem[a0 + half], IntF::ld(tw, m + i), K);
      }
      __syncthreads();
      half <<= 1;
    }
    for (u32 a = threadIdx.x; a < n; a += blockDim.x)
      out(a, mul_shoup(smem[a], P.n_inv, P.n_inv_shoup, P.q));
  }
}

}  // namespace lcl
