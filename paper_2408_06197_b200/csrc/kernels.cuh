// Tensor, accumulation and key inner-product kernels for the server path.
#pragma once

#include "common.cuh"

namespace lcl {

// ------------------------------------------------------------------------
// Pairwise lazy accumulation (distance.cpp:107-127 lazy branch):
//   for every pair (i, j) and chunk c:  e = a_i[c] - a_j[c]  (hsub)
//   d0 += e0^2, d1 += 2 e0 e1, d2 += e1^2                   (hsquare + lazy_accumulate)
// All C chunks of all pairs are folded into split-23 partial sums in
// registers and reduced once, so the ternary accumulator is written once and
// every client word is read once per CTA (client tile staged in shared memory
// and reused by every pair in the CTA).
//
// CTA: 32 consecutive slots of one limb row r; warp w, lane e handles PP pairs
// of that slot. Grid: x = m * N / 32 slot tiles, y = pair groups. The client
// tile of chunk c + STAGES - 1 streams into shared memory (cp.async) while
// chunk c is being accumulated.
// clients: [n][C][2][m][N]; tern out: [pairs][3][m][N] (pair p at out + (p - p0) * 3mN).
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}

// Tile = TE consecutive slots of one limb row r for a group of pairs; thread
// (pair, eg) owns EPT slots of one pair. Every client word of the tile is
// streamed into shared memory once per pair group (16-byte cp.async, STAGES
// deep; load addresses computed once) and read by all pairs in it, so for up
// to 256 pairs the client data crosses HBM exactly once.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const u32 s = (u32)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

template <int TE, int EPT, int STAGES>
__global__ void __launch_bounds__(512)
    pair_accumulate(const u64* __restrict__ clients, u32 n, u32 c_begin, u32 c_end,
                    u32 chunks_total, u32 m, u32 logn, const u32* __restrict__ pairs,
                    u32 p_begin, u32 p_end, u32 pairs_per_cta, u64* __restrict__ tern,
                    int accumulate, const PrimeConst* __restrict__ primes) {
  static_assert(EPT % 2 == 0, "slots are read from shared memory in 16-byte pairs");
  constexpr int TPP = TE / EPT;    // threads per pair
  constexpr int CS = 2 * TE + 2;   // words per client in the tile (16-B aligned, banks spread)
  constexpr int V = 2 * TE / 2;    // 16-byte vectors per client per chunk
  constexpr int MAXV = 4;          // vectors per thread (n * V <= MAXV * blockDim)
  extern __shared__ u64 tile[];    // [STAGES][n][CS]
  const u32 N = 1u << logn;
  const u32 tiles_per_row = N / TE;
  const u32 r = blockIdx.x / tiles_per_row;
  const u32 a0 = (blockIdx.x - r * tiles_per_row) * TE;
  const PrimeConst P = primes[r];
  const u64 q = P.q;
  const u64 ct_words = 2ull * m * N;
  const u32 tw = n * CS;
  const u32 p = p_begin + blockIdx.y * pairs_per_cta + threadIdx.x / TPP;
  const u32 eg = threadIdx.x % TPP;
  const bool valid = threadIdx.x / TPP < pairs_per_cta && p < p_end;
  const u32 pk = valid ? __ldg(pairs + p) : 0u;
  const u32 oi = (pk & 0xFFFFu) * CS + eg * EPT, oj = (pk >> 16) * CS + eg * EPT;

  // this thread's 16-byte load slots: (global address at chunk 0, smem word)
  const u64* gsrc[MAXV];
  u32 soff[MAXV];
  u32 nv = 0;
#pragma unroll
  for (int s = 0; s < MAXV; ++s) {
    const u32 v = threadIdx.x + s * blockDim.x;
    gsrc[s] = nullptr;
    soff[s] = 0;
    if (v < n * V) {
      const u32 cl = v / V, w = (v - cl * V) * 2, h = w / TE, e = w - h * TE;
      gsrc[s] = clients + (u64)cl * chunks_total * ct_words + (u64)h * m * N + (u64)r * N + a0 + e;
      soff[s] = cl * CS + w;
      nv = s + 1;
    }
  }
  auto issue = [&](u32 c, u32 stage) {
    if (c < c_end) {
#pragma unroll
      for (int s = 0; s < MAXV; ++s)
        if (s < (int)nv) cp_async16(tile + stage * tw + soff[s], gsrc[s] + (u64)c * ct_words);
    }
    cp_async_commit();  // empty groups keep the wait count uniform
  };

  // A00 / A11 hold e^2 with the cross term accumulated once (lo * hi) and
  // doubled in the final reduction; A01 holds e0 * e1.
  Acc3 A00[EPT], A01[EPT], A11[EPT];
#pragma unroll
  for (int t = 0; t < EPT; ++t) {
    A00[t].zero();
    A01[t].zero();
    A11[t].zero();
  }
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(c_begin + s, s);
  // One barrier per chunk: after it every thread has finished chunk c - 1, so
  // its stage can be refilled with chunk c + STAGES - 1 while c is consumed.
  u32 stage = 0;
  for (u32 c = c_begin; c < c_end; ++c) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue(c + STAGES - 1, stage == 0 ? STAGES - 1 : stage - 1);
    const u64* tl = tile + stage * tw;
#pragma unroll
    for (int t = 0; t < EPT; t += 2) {
      const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(tl + oi + t);
      const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(tl + oi + TE + t);
      const ulonglong2 y0 = *reinterpret_cast<const ulonglong2*>(tl + oj + t);
      const ulonglong2 y1 = *reinterpret_cast<const ulonglong2*>(tl + oj + TE + t);
      {
        const Split e0 = split23(x0.x - y0.x + q), e1 = split23(x1.x - y1.x + q);
        A00[t].sqh(e0);
        A01[t].mac(e0, e1);
        A11[t].sqh(e1);
      }
      {
        const Split e0 = split23(x0.y - y0.y + q), e1 = split23(x1.y - y1.y + q);
        A00[t + 1].sqh(e0);
        A01[t + 1].mac(e0, e1);
        A11[t + 1].sqh(e1);
      }
    }
    stage = stage + 1 == STAGES ? 0 : stage + 1;
  }
  if (!valid) return;
#pragma unroll
  for (int t = 0; t < EPT; ++t) {
    u64* o = tern + (u64)(p - p_begin) * 3 * m * N + (u64)r * N + a0 + eg * EPT + t;
    u64 d0 = A00[t].reduce_sq(P);
    u64 d1 = A01[t].reduce(P);
    d1 = add_mod(d1, d1, q);
    u64 d2 = A11[t].reduce_sq(P);
    if (accumulate) {
      d0 = add_mod(d0, o[0], q);
      d1 = add_mod(d1, o[(u64)m * N], q);
      d2 = add_mod(d2, o[2ull * m * N], q);
    }
    o[0] = d0;
    o[(u64)m * N] = d1;
    o[2ull * m * N] = d2;
  }
}

// FP64-pipe form of the same accumulation, for q-chains below 2^44. B200
// retires 64 DFMA/clk/SM but only 32 IMAD.WIDE/clk/SM, so the products run
// on the FP64 pipe. A residue x < 2^44 is read as the double X = 2^52 + x by
// OR-ing the exponent into its high word (no conversion instruction), so
// e = X_i - X_j is exact. Every product p = a * b (|p| < 2^88) is split
// exactly on a 2^44 grid with one FMA against M = 1.5 * 2^96:
//   t = fl(p + M), hi = t - M = H * 2^44 (|H| <= 2^44), lo = fma(a, b, -hi)
// (|lo| <= 2^43, exact), and H, lo go to two double accumulators that stay
// exact integers (< 2^53) for 256 chunks; the launcher splits longer chunk
// ranges and re-enters with accumulate = 1. 2 DADD + 3 x 5 FP64 ops per slot
// and pair, 6 accumulators. The words are the integer kernel's, reduced mod q
// once at the end.
__device__ __forceinline__ u64 dmodq(double v, u64 q, const PrimeConst& P) {
  const long long i = __double2ll_rn(v);  // exact: |v| < 2^53 is an integer
  if (i >= 0) return reduce64((u64)i, P);
  const u64 r = reduce64((u64)(-i), P);
  return r ? q - r : 0;
}

// A thread owns one pair for the TE slots of its tile. Pairs are assigned to
// threads by a host schedule (sched[k] = (i | j << 16, output index)) that
// puts clients of distinct shared-memory bank groups in every quarter warp,
// so the 16-byte tile reads are conflict-free.
// W > 1 (at most 32 pairs per CTA): the CTA's tile is W * TE slots wide and
// warp w owns slots [w TE, (w + 1) TE) of it for the same pairs, so every
// (client, poly) piece copied per chunk is W * 64 bytes: 64-byte pieces cap
// the staging at ~3 TB/s, 256-byte ones reach ~7 TB/s
// (tools/microbench/stride_probe.cu) -- the case of a host-round group of
// one client, whose few pairs leave the FP64 pipe idle.
template <int TE, int STAGES, int MAXT, int MINB, bool PF, int W = 1>
__global__ void __launch_bounds__(MAXT, MINB)
    pair_accumulate_f64(const u64* __restrict__ clients, u32 n, u32 c_begin, u32 c_end,
                        u32 chunks_total, u32 m, u32 logn, const uint2* __restrict__ sched,
                        u32 pairs, u32 groups, u32 pairs_per_cta, u64* __restrict__ tern,
                        int accumulate, const PrimeConst* __restrict__ primes,
                        const unsigned short* __restrict__ clist, u32 nl) {
  static_assert(TE % 2 == 0, "slots are read from shared memory in 16-byte pairs");
  constexpr int CS = 2 * TE + 2;  // words per client: CS / 2 odd spreads clients over bank groups
  extern __shared__ u64 tile[];   // [STAGES][W][nl][CS]
  const u32 N = 1u << logn;
  const u32 tiles_per_row = N / (TE * W);
  const u32 g = blockIdx.x % groups;
  const u32 tix = blockIdx.x / groups;
  const u32 r = tix / tiles_per_row;
  const u32 a0 = (tix - r * tiles_per_row) * (TE * W);
  const u32 sub = W > 1 ? threadIdx.x / 32 : 0;     // the thread's TE-slot sub-tile
  const u32 pt = W > 1 ? threadIdx.x % 32 : threadIdx.x;  // its pair within the CTA
  const u64 ct_words = 2ull * m * N;
  // clients staged by this CTA: all n (clist == nullptr), or the nl clients
  // of its client-blocked pair group, clist[g * nl ..]
  if (!clist) nl = n;
  const unsigned short* gl = clist ? clist + (size_t)g * nl : nullptr;
  const u32 tw = W * nl * CS;
  const u32 k = g * pairs_per_cta + pt;
  // schedule entries with .y == ~0 pad a group to pairs_per_cta
  const uint2 sk = pt < pairs_per_cta && k < pairs ? __ldg(sched + k) : make_uint2(0u, ~0u);
  const bool valid = sk.y != ~0u;
  const u32 oi = (sub * nl + (sk.x & 0xFFFFu)) * CS, oj = (sub * nl + (sk.x >> 16)) * CS;

  // chunk copies: nl * TE 16-byte vectors, vector v by thread v mod blockDim.
  // The first vector's addresses are computed once (every thread has at most
  // one when nl * TE <= blockDim, the common case); further ones per chunk.
  const u64* cbase = clients + (u64)r * N + a0;
  // vector v: client cl, poly h, word x of the poly's W * TE-word piece
  // (consecutive v read consecutive 16 bytes), parked in sub-tile x / TE
  auto vec_src = [&](u32 v, u32& soff) {
    const u32 cl = v / (W * TE), rest = (v % (W * TE)) * 2;
    const u32 h = rest / (W * TE), x = rest % (W * TE), ws = x / TE, e = x % TE;
    soff = (ws * nl + cl) * CS + h * TE + e;
    const u32 gc = gl ? (u32)__ldg(gl + cl) : cl;
    return cbase + (u64)gc * chunks_total * ct_words + (u64)h * m * N + x;
  };
  const bool has0 = threadIdx.x < nl * TE * W;
  u32 soff0 = 0;
  const u64* src0 = has0 ? vec_src(threadIdx.x, soff0) : cbase;
  auto issue = [&](u32 c, u32 stage) {
    if (c < c_end) {
      if (has0) cp_async16(tile + stage * tw + soff0, src0 + (u64)c * ct_words);
      for (u32 v = threadIdx.x + blockDim.x; v < nl * TE * W; v += blockDim.x) {
        u32 so;
        const u64* g = vec_src(v, so);
        cp_async16(tile + stage * tw + so, g + (u64)c * ct_words);
      }
    }
    cp_async_commit();
  };

  // per slot: (H, lo) accumulators of e0^2, e0 e1, e1^2
  double S[TE][6];
#pragma unroll
  for (int t = 0; t < TE; ++t)
#pragma unroll
    for (int q = 0; q < 6; ++q) S[t][q] = 0.0;
  constexpr double kM = 118842243771396506390315925504.0;  // 1.5 * 2^96
  constexpr double kInv44 = 1.0 / 17592186044416.0;        // 2^-44
  auto as_d = [](u64 x) { return __longlong_as_double((long long)(x | 0x4330000000000000ull)); };
  auto prod = [&](double a, double b, double& accH, double& accL) {
    const double hi = __dadd_rn(__fma_rn(a, b, kM), -kM);
    accL = __dadd_rn(accL, __fma_rn(a, b, -hi));
    accH = __fma_rn(hi, kInv44, accH);
  };
  // Chunk c + 1's words are read from shared memory into registers while
  // chunk c is multiplied, so shared-memory latency hides behind a whole
  // chunk of FP64 work; one barrier per chunk recycles the ring stage.
  static_assert(STAGES >= 3, "the register prefetch runs one chunk ahead of the math");
  ulonglong2 cur[4][TE / 2], nxt[4][TE / 2];
  auto load = [&](u32 stage, ulonglong2 (&v)[4][TE / 2]) {
    const u64* tl = tile + stage * tw;
#pragma unroll
    for (int t = 0; t < TE / 2; ++t) {
      v[0][t] = *reinterpret_cast<const ulonglong2*>(tl + oi + 2 * t);
      v[1][t] = *reinterpret_cast<const ulonglong2*>(tl + oi + TE + 2 * t);
      v[2][t] = *reinterpret_cast<const ulonglong2*>(tl + oj + 2 * t);
      v[3][t] = *reinterpret_cast<const ulonglong2*>(tl + oj + TE + 2 * t);
    }
  };
  auto math = [&](const ulonglong2 (&v)[4][TE / 2]) {
#pragma unroll
    for (int t = 0; t < TE / 2; ++t) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double e0 = __dadd_rn(as_d(u ? v[0][t].y : v[0][t].x), -as_d(u ? v[2][t].y : v[2][t].x));
        const double e1 = __dadd_rn(as_d(u ? v[1][t].y : v[1][t].x), -as_d(u ? v[3][t].y : v[3][t].x));
        double* a = S[2 * t + u];
        prod(e0, e0, a[0], a[1]);
        prod(e0, e1, a[2], a[3]);
        prod(e1, e1, a[4], a[5]);
      }
    }
  };
  if constexpr (!PF) {
    // two chunks per barrier: chunk k lives in stage k % STAGES; the prologue
    // fills STAGES - 2 stages, and each iteration refills the two stages the
    // previous one consumed with chunks c + STAGES - 2 and c + STAGES - 1
    static_assert(STAGES >= 4, "two chunks in flight per iteration");
#pragma unroll
    for (int s = 0; s < STAGES - 2; ++s) issue(c_begin + s, s);
    u32 stage = 0;  // stage of chunk c
    u32 c = c_begin;
    for (; c + 2 <= c_end; c += 2) {
      cp_async_wait<STAGES - 4>();
      __syncthreads();
      const u32 s1 = stage + 1 == STAGES ? 0 : stage + 1;
      issue(c + STAGES - 2, stage >= 2 ? stage - 2 : stage + STAGES - 2);
      issue(c + STAGES - 1, stage >= 1 ? stage - 1 : STAGES - 1);
      ulonglong2 v[4][TE / 2];
      load(stage, v);
      math(v);
      load(s1, v);
      math(v);
      stage = s1 + 1 == STAGES ? 0 : s1 + 1;
    }
    if (c < c_end) {  // odd tail
      cp_async_wait<0>();
      __syncthreads();
      ulonglong2 v[4][TE / 2];
      load(stage, v);
      math(v);
    }
  } else {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue(c_begin + s, s);
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    load(0, cur);
    u32 stage = 0;
    for (u32 c = c_begin; c < c_end; ++c) {
      cp_async_wait<STAGES - 3>();  // chunk c + 1 has landed
      __syncthreads();              // and every thread holds chunk c in registers
      issue(c + STAGES - 1, stage == 0 ? STAGES - 1 : stage - 1);  // chunk c - 1's stage
      const u32 ns = stage + 1 == STAGES ? 0 : stage + 1;
      if (c + 1 < c_end) load(ns, nxt);
      math(cur);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int t = 0; t < TE / 2; ++t) cur[k][t] = nxt[k][t];
      stage = ns;
    }
  }
  if (!valid) return;
  const PrimeConst P = primes[r];
  const u64 q = P.q;
  const u64 w44 = reduce64(1ull << 44, P);
  auto combine = [&](double h, double l) {  // h * 2^44 + l  (mod q)
    return add_mod(mul_mod(dmodq(h, q, P), w44, P), dmodq(l, q, P), q);
  };
  u64* ob = tern + (u64)sk.y * 3 * m * N + (u64)r * N + a0 + sub * TE;
#pragma unroll
  for (int t = 0; t < TE; ++t) {
    u64* o = ob + t;
    u64 d0 = combine(S[t][0], S[t][1]);
    u64 d1 = combine(S[t][2], S[t][3]);
    d1 = add_mod(d1, d1, q);  // hsquare's 2 c0 c1
    u64 d2 = combine(S[t][4], S[t][5]);
    if (accumulate) {
      d0 = add_mod(d0, o[0], q);
      d1 = add_mod(d1, o[(u64)m * N], q);
      d2 = add_mod(d2, o[2ull * m * N], q);
    }
    o[0] = d0;
    o[(u64)m * N] = d1;
    o[2ull * m * N] = d2;
  }
}

// ------------------------------------------------------------------------
// Masked aggregation tensor (aggregation.cpp:205-219): per chunk ch,
//   sum_i hmult_triple(w_i[ch], sel_i) with Karatsuba d1 = (w0+w1)(s0+s1) - d0 - d2,
// lazily accumulated over the clients in split-23 sums, reduced once.
// A thread owns 2 consecutive slots of one limb of one chunk (16-byte loads)
// and walks clients [i0, i1); the (w0, w1, s0, s1) vectors of client
// i + STAGES - 1 are copied into a private shared-memory ring (cp.async, no
// barrier: a thread only reads what it copied) while client i is
// accumulated, so HBM latency is hidden by the copy ring rather than by
// registers. Selectors are re-read per chunk from L2 (n * ct, small). The sum
// is linear, so client ranges accumulate (accumulate = 1 adds mod q to tern).
// clients: [n][C][2][m][N]; sel: [n][2][m][N]; tern: [chunks][3][m][N].
template <int STAGES>
__global__ void __launch_bounds__(256)
    aggregate_stream(const u64* __restrict__ clients, const u64* __restrict__ sel, u32 i0, u32 i1,
                     u32 chunks_total, u32 c_begin, u32 chunks, u32 m, u32 logn,
                     u64* __restrict__ tern, int accumulate, const PrimeConst* __restrict__ primes) {
  extern __shared__ ulonglong2 ring[];  // [STAGES][4][blockDim]
  const u32 N = 1u << logn;
  // chunk-fastest CTA order: the `chunks` CTAs of one slot block run back to
  // back, so its selector words come from L2 instead of being re-read from
  // HBM once per chunk (the client stream would evict them)
  const u32 ch = blockIdx.x % chunks;
  const u32 rem = ((blockIdx.x / chunks) * blockDim.x + threadIdx.x) * 2;
  const u32 r = rem >> logn, a = rem & (N - 1);
  const PrimeConst P = primes[r];
  const u64 q = P.q;
  const u64 slots = (u64)m * N;
  const u64 ct_words = 2ull * m * N;
  const u64 client_stride = (u64)chunks_total * ct_words;
  const u64* wp = clients + (u64)(c_begin + ch) * ct_words + (u64)r * N + a;
  const u64* sp = sel + (u64)r * N + a;
  const u32 bd = blockDim.x;
  ulonglong2* my = ring + threadIdx.x;
  auto issue = [&](u32 i, u32 st) {
    if (i < i1) {
      ulonglong2* d = my + st * 4 * bd;
      const u64* w = wp + (u64)i * client_stride;
      const u64* s = sp + (u64)i * ct_words;
      cp_async16(d, w);
      cp_async16(d + bd, w + slots);
      cp_async16(d + 2 * bd, s);
      cp_async16(d + 3 * bd, s + slots);
    }
    cp_async_commit();
  };
  Acc3 D0[2], D1[2], D2[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    D0[k].zero();
    D1[k].zero();
    D2[k].zero();
  }
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(i0 + s, s);
  u32 st = 0;
  for (u32 i = i0; i < i1; ++i) {
    cp_async_wait<STAGES - 2>();
    const ulonglong2* d = my + st * 4 * bd;
    const ulonglong2 w0 = d[0], w1 = d[bd], s0 = d[2 * bd], s1 = d[3 * bd];
    issue(i + STAGES - 1, st == 0 ? STAGES - 1 : st - 1);
    D0[0].mac(split23(w0.x), split23(s0.x));
    D2[0].mac(split23(w1.x), split23(s1.x));
    D1[0].mac(split23(w0.x + w1.x), split23(s0.x + s1.x));
    D0[1].mac(split23(w0.y), split23(s0.y));
    D2[1].mac(split23(w1.y), split23(s1.y));
    D1[1].mac(split23(w0.y + w1.y), split23(s0.y + s1.y));
    st = st + 1 == STAGES ? 0 : st + 1;
  }
  u64* o = tern + (u64)ch * 3 * slots + (u64)r * N + a;
  ulonglong2 o0, o1, o2;
  o0.x = D0[0].reduce(P);
  o2.x = D2[0].reduce(P);
  o1.x = sub_mod(sub_mod(D1[0].reduce(P), o0.x, q), o2.x, q);
  o0.y = D0[1].reduce(P);
  o2.y = D2[1].reduce(P);
  o1.y = sub_mod(sub_mod(D1[1].reduce(P), o0.y, q), o2.y, q);
  if (accumulate) {
    const ulonglong2 p0 = *reinterpret_cast<const ulonglong2*>(o);
    const ulonglong2 p1 = *reinterpret_cast<const ulonglong2*>(o + slots);
    const ulonglong2 p2 = *reinterpret_cast<const ulonglong2*>(o + 2 * slots);
    o0.x = add_mod(o0.x, p0.x, q);
    o0.y = add_mod(o0.y, p0.y, q);
    o1.x = add_mod(o1.x, p1.x, q);
    o1.y = add_mod(o1.y, p1.y, q);
    o2.x = add_mod(o2.x, p2.x, q);
    o2.y = add_mod(o2.y, p2.y, q);
  }
  *reinterpret_cast<ulonglong2*>(o) = o0;
  *reinterpret_cast<ulonglong2*>(o + slots) = o1;
  *reinterpret_cast<ulonglong2*>(o + 2 * slots) = o2;
}

// ------------------------------------------------------------------------
// Key inner product (ckks.cpp:490-518 without the ModDown):
//   acc_x[b][r][a] = sum_j digit_j[b][r][g(a)] * key_x[j][kr][a],  g = perm or identity
// digits: [B][M][M+1][N]; key: [full][2][full+1][N]; acc: [B][2][M+1][N].
// A thread owns one slot of one target row for IB consecutive ciphertexts:
// the 2M key words stay in registers and are reused IB times; grid.y walks
// the batch, so every key word is read from HBM once per launch (L2 serves
// the other item blocks). Products < 2^108 are summed exactly in 128 bits.
template <int M, int IB>
__global__ void __launch_bounds__(256)
    ks_inner_product(const u64* __restrict__ digits, u32 B, const u64* __restrict__ key,
                     u32 full, const u32* __restrict__ perm, u64* __restrict__ acc, u32 logn,
                     const PrimeConst* __restrict__ primes) {
  const u32 N = 1u << logn;
  const u32 gid = blockIdx.x * blockDim.x + threadIdx.x;
  const u32 r = gid >> logn, a = gid & (N - 1);
  if (r > (u32)M) return;
  const u32 b0 = blockIdx.y * IB;
  const u32 kr = r < (u32)M ? r : full;
  const PrimeConst P = primes[kr];
  const u64 kstride = (u64)(full + 1) * N;
  u64 k0[M], k1[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    k0[j] = __ldg(key + (2ull * j) * kstride + (u64)kr * N + a);
    k1[j] = __ldg(key + (2ull * j + 1) * kstride + (u64)kr * N + a);
  }
  const u32 g = perm ? __ldg(perm + a) : a;
  const u64 dstride = (u64)(M + 1) * N;
#pragma unroll 2
  for (int i = 0; i < IB; ++i) {
    const u32 b = b0 + i;
    if (b >= B) break;
    const u64* d = digits + (u64)b * M * dstride + (u64)r * N + g;
    u64 v[M];
#pragma unroll
    for (int j = 0; j < M; ++j) v[j] = __ldg(d + j * dstride);
    u64 l0 = 0, h0 = 0, l1 = 0, h1 = 0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      mac128(l0, h0, v[j], k0[j]);
      mac128(l1, h1, v[j], k1[j]);
    }
    u64* o = acc + (u64)b * 2 * dstride + (u64)r * N + a;
    o[0] = reduce128(l0, h0, P);
    o[dstride] = reduce128(l1, h1, P);
  }
}

// ------------------------------------------------------------------------
// ct x ct tensor (ckks.cpp:417-451) over B pairs of ciphertexts [B][2][m][N]:
// hmult_triple (Karatsuba: d1 = (a0 + a1)(b0 + b1) - d0 - d2) or, when
// b == a, hsquare (d1 = 2 a0 a1); both are the same residues as the
// schoolbook product. out: [B][3][m][N].
__global__ void __launch_bounds__(256)
    ct_tensor(const u64* __restrict__ a, const u64* __restrict__ b, u32 B, u32 m, u32 logn,
              u64* __restrict__ out, const PrimeConst* __restrict__ primes) {
  const u32 N = 1u << logn;
  const u64 slots = (u64)m * N;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)B * slots) return;
  const u64 item = gid / slots, s = gid - item * slots;
  const PrimeConst P = primes[(u32)(s >> logn)];
  const u64 q = P.q;
  const u64 a0 = a[item * 2 * slots + s], a1 = a[item * 2 * slots + slots + s];
  u64* o = out + item * 3 * slots + s;
  if (a == b) {
    const u64 d0 = mul_mod(a0, a0, P), d2 = mul_mod(a1, a1, P);
    const u64 x = mul_mod(a0, a1, P);
    o[0] = d0;
    o[slots] = add_mod(x, x, q);
    o[2 * slots] = d2;
    return;
  }
  const u64 b0 = b[item * 2 * slots + s], b1 = b[item * 2 * slots + slots + s];
  const u64 d0 = mul_mod(a0, b0, P), d2 = mul_mod(a1, b1, P);
  const u64 k = mul_mod(add_mod(a0, a1, q), add_mod(b0, b1, q), P);
  o[0] = d0;
  o[slots] = sub_mod(sub_mod(k, d0, q), d2, q);
  o[2 * slots] = d2;
}

// Sum of `shards` partial ternaries (u64 words, each < q, added as plain
// integers by an NCCL SUM: < shards * q < 2^64) reduced mod q in place;
// tern [P][3][m][N], row prime = limb index.
__global__ void __launch_bounds__(256)
    reduce_partials(u64* __restrict__ tern, u64 words, u32 m, u32 logn,
                    const PrimeConst* __restrict__ primes) {
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= words) return;
  const u32 limb = (u32)((gid >> logn) % m);
  tern[gid] = reduce64(tern[gid], primes[limb]);
}

// ------------------------------------------------------------------------
// LCLT wire format (CkksContext::serialize / deserialize, ckks.cpp:614-678):
// a 13-byte header (magic "LCLT", u16 version, u32 ring degree, u8 level,
// u8 scale bits, u8 limb count) then the c0 rows and the c1 rows as
// little-endian u64 -- so every payload word sits 5 bytes off an 8-byte
// boundary. Blob (r, c) of an [rows][cols] batch starts at byte
// (r * cols + c) * stride of `blobs` (the host layout, copied verbatim);
// ciphertext (r, c) lands at (r * cols + c) * 2 m N words of `out`. Items
// (r, c0 .. c1) of rows r0 .. r1 are unpacked: each thread funnel-shifts two
// aligned 8-byte loads per word, checks the residue against its prime
// (deserialize's "residue outside its modulus") and records the first bad
// blob in *err (atomicMin over a word initialised to UINT_MAX).
__global__ void __launch_bounds__(256)
    lclt_unpack(const u8* __restrict__ blobs, u64 stride, u32 cols, u32 r0, u32 c0, u32 ncols,
                u32 m, u32 logn, u64* __restrict__ out, u32* __restrict__ err,
                const PrimeConst* __restrict__ primes) {
  const u64 W = 2ull * m << logn;
  const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= W) return;
  const u32 r = r0 + blockIdx.y / ncols, c = c0 + blockIdx.y % ncols;
  const u64 item = (u64)r * cols + c;
  const u64 byte = item * stride + 13 + 8 * k;
  const u64* w = reinterpret_cast<const u64*>(blobs) + (byte >> 3);
  const u32 sh = (u32)(byte & 7) * 8;
  const u64 lo = __ldg(w);
  const u64 v = sh ? (lo >> sh) | (__ldg(w + 1) << (64 - sh)) : lo;
  const u32 limb = (u32)((k >> logn) % m);
  if (v >= primes[limb].q) atomicMin(err, (u32)item);
  out[item * W + k] = v;
}

// serialize (ckks.cpp:614-638): ciphertexts [items][2][m][N] -> blobs at
// `stride` bytes with the LCLT header; one thread per 8 payload bytes,
// thread 0 of each blob also writes the header. Byte stores (the payload is
// 5 bytes off alignment); the blob bytes leave the device with one copy.
__global__ void __launch_bounds__(256)
    lclt_pack(const u64* __restrict__ ct, u32 m, u32 logn, u32 level, u32 scale_bits,
              u64 stride, u8* __restrict__ blobs) {
  const u64 W = 2ull * m << logn;
  const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 item = blockIdx.y;
  u8* b = blobs + item * stride;
  if (k == 0) {
    const u32 n = 1u << logn;
    const u8 hdr[13] = {'L', 'C', 'L', 'T', 1, 0, (u8)n, (u8)(n >> 8), (u8)(n >> 16),
                        (u8)(n >> 24), (u8)level, (u8)scale_bits, (u8)m};
#pragma unroll
    for (int i = 0; i < 13; ++i) b[i] = hdr[i];
  }
  if (k >= W) return;
  const u64 v = __ldg(ct + item * W + k);
  u8* p = b + 13 + 8 * k;
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = (u8)(v >> (8 * i));
}

// ------------------------------------------------------------------------
// DistanceMode::row_sums (distance.cpp:287-298): row i of the matrix is the
// sum of the n - 1 pair ciphertexts that contain client i. pairs: [P][W]
// words in (i<j) row-major order, W = 2 m N; rows: [n][W]. Modular addition
// is exact, so the sum equals the reference's left-to-right hadd chain word
// for word. Two 64-bit words per thread (128-bit loads and stores).
__global__ void __launch_bounds__(256)
    pair_row_sums(const u64* __restrict__ pairs, u32 n, u32 m, u32 logn, u64* __restrict__ rows,
                  const PrimeConst* __restrict__ primes) {
  const u64 W = 2ull * m << logn;
  const u64 gid = ((u64)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  const u32 i = blockIdx.y;
  if (gid >= W) return;
  const u32 limb = (u32)((gid >> logn) % m);
  const u64 q = primes[limb].q;
  u64 a0 = 0, a1 = 0;
  for (u32 o = 0; o < n; ++o) {
    if (o == i) continue;
    const u32 lo = o < i ? o : i, hi = o < i ? i : o;
    // index of (lo, hi) in the row-major i<j order
    const u64 p = (u64)lo * (2ull * n - lo - 1) / 2 + (hi - lo - 1);
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(pairs + p * W + gid));
    a0 = add_mod(a0, v.x, q);
    a1 = add_mod(a1, v.y, q);
  }
  *reinterpret_cast<ulonglong2*>(rows + (u64)i * W + gid) = make_ulonglong2(a0, a1);
}

// ------------------------------------------------------------------------
// ct x pt (ckks.cpp:549-558): out[b][x][i][a] = ct[b][x][i][a] * pt[i][a].
__global__ void __launch_bounds__(256)
    mult_plain(const u64* __restrict__ ct, const u64* __restrict__ pt, u32 B, u32 m, u32 logn,
               u64* __restrict__ out, const PrimeConst* __restrict__ primes) {
  const u32 N = 1u << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 total = (u64)B * 2 * m * N;
  if (gid >= total) return;
  const u32 a = (u32)(gid & (N - 1));
  const u32 i = (u32)((gid >> logn) % m);
  const PrimeConst P = primes[i];
  out[gid] = mul_mod(__ldg(ct + gid), __ldg(pt + (u64)i * N + a), P);
}

// Elementwise add / sub over ciphertext batches with RowMap addressing.
template <bool SUB>
__global__ void __launch_bounds__(256)
    rows_addsub(const __grid_constant__ RowMap out, const __grid_constant__ RowMap a,
                const __grid_constant__ RowMap b, u32 rows, u32 logn,
                const PrimeConst* __restrict__ primes) {
  const u32 N = 1u << logn;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (u64)rows * N) return;
  const u32 r = (u32)(gid >> logn), k = (u32)(gid & (N - 1));
  const u64 q = primes[row_prime(out, r)].q;
  const u64 x = row_ptr(a, r)[k], y = row_ptr(b, r)[k];
  row_ptr(out, r)[k] = SUB ? sub_mod(x, y, q) : add_mod(x, y, q);
}

// ------------------------------------------------------------------------
// Integer roofline probe: independent chains of the forward NTT butterfly
// (Shoup product + add / offset-sub, the instruction mix of ct_bfly) on
// register-resident data. 16 independent butterflies per thread per
// iteration; the result is folded into one store so nothing is dead code.
__global__ void __launch_bounds__(256) peak_butterfly(u64* __restrict__ sink, u32 iters, u64 q,
                                                      u64 w, u64 ws) {
  u64 x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (threadIdx.x * 131 + i * 977 + blockIdx.x) % q;
  const u64 two_q = 2 * q;
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      // the forward butterfly of ntt.cuh (values wrap here; only the
      // instruction stream matters for the probe)
      const u64 t = mul_shoup_lazy4(x[2 * i + 1], w, ws, q);
      const u64 a = x[2 * i];
      x[2 * i] = a + t;
      x[2 * i + 1] = a + (2 * two_q - t);
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s ^= x[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Same probe for the FP64-pipe butterfly of ntt.cuh (FpF::ct: f_mulmod + two
// DADD on exact integer-valued doubles), the field of the q-chain rows.
__global__ void __launch_bounds__(256) peak_butterfly_f64(u64* __restrict__ sink, u32 iters,
                                                          double q, double w, double wq) {
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (double)((threadIdx.x * 131 + i * 977 + blockIdx.x) % 100003);
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double t = f_mulmod(x[2 * i + 1], w, wq, q);
      const double a = x[2 * i];
      x[2 * i] = __dadd_rn(a, t);
      x[2 * i + 1] = __dadd_rn(a, -t);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += x[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = (u64)__double_as_longlong(s);
}

}  // namespace lcl
