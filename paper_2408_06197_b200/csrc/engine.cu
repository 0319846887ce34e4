// Host runtime + C-ABI of the B200-native Lancelot server path.
//
// Everything below the C-ABI is native: basis construction (prime search,
// psi, twiddle and Shoup tables), key residency in HBM, a grow-only device
// workspace, and the batched orchestration of the reference's server
// functions as level-synchronous kernel sequences on one CUDA stream.
//
// Reference call structure mirrored here (paths under /root/reference/proj/core):
//   build_distance_matrix      distance.cpp:242-300
//   encrypted_pairwise_distance distance.cpp:107-142
//   slot_reduce                distance.cpp:214-240
//   masked_aggregate           aggregation.cpp:188-229
//   relinearize / rescale / rotate / hoisted_rotations   ckks.cpp:522-612
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <utility>
#include <random>
#include <thread>
#include <tuple>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lancelot_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "decode.cuh"
#include "encrypt.cuh"
#include "ntt.cuh"

using namespace lcl;

typedef unsigned __int128 u128;

namespace {

// CTAs/SM bound of ntt_blk_fwd<DivRoundInvStore>. At 16 (64 registers) it
// spills 276 B per thread; 12 (80 registers, 12 B spill) and 10 measured
// slower at cfg3 (9.51 / 10.26 vs 9.25 ms): the spills stay in L1.
// Single rotations through modup_ip_hoist (ns = 1: digits parked in shared
// memory, register accumulators) instead of modup_ip_blk: measured 11.81 vs
// 10.44 ms at cfg3 (10 instead of 16 warps/SM), so off.
#ifndef LCL_ROT_HOIST
#define LCL_ROT_HOIST 0
#endif
// modup_ip_blk as two field-specialised launches (special target on the
// integer pipe, then the q targets on the FP64 pipe) instead of one kernel
// carrying both fields' code: measured neutral at cfg3 (10.57 vs 10.55 ms),
// so the single launch stays the default.
#ifndef LCL_MODUP_SPLIT
#define LCL_MODUP_SPLIT 0
#endif
// Divide-and-round block passes with TMA-staged operands (ntt_blk_fwd_dr_tma)
// and their CTAs/SM bound (33 KB of shared memory per CTA: at most 6).
// Measured at cfg3: <divround+inv> 7.99 -> 13.90 ms, <divround> 4.61 -> 7.89
// (12 warps/SM instead of 32: the staging buffers cost more occupancy than
// the early loads buy), so the register-load kernel stays the default.
#ifndef LCL_DR_TMA
#define LCL_DR_TMA 0
#endif
#ifndef LCL_DR_MINB
#define LCL_DR_MINB 6
#endif
// CTAs/SM bound of the fused column pass at E = 16. With the source tile
// parked in shared memory (LCL_COL_VSMEM, 64 KB per CTA) 3 CTAs fit, at 80
// registers and no spill: cfg3 column passes 17.43 -> 16.98 ms against
// 4 CTAs at 64 registers with 900 B of spill loads per thread (2 CTAs at
// 128 registers: 17.77 ms).
#ifndef LCL_COL_MINB
#define LCL_COL_MINB 3
#endif
#ifndef LCL_INV_MINB
#define LCL_INV_MINB 16
#endif

// ------------------------------------------------------------ errors
thread_local std::string g_last_error;

struct Status {
  int code;
  std::string msg;
};

struct LclError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw LclError{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(LCL_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void need(bool ok, int code, const char* msg) {
  if (!ok) fail(code, msg);
}

// ------------------------------------------------------------ host modular math
// Setup-time only (basis construction); restates modmath.cpp:24-132.
u64 h_mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
u64 h_powmod(u64 b, u64 e, u64 q) {
  u64 r = 1;
  b %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, b, q);
    b = h_mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}
u64 h_invmod(u64 a, u64 q) { return h_powmod(a % q, q - 2, q); }
bool h_is_prime(u64 n) {
  static const u64 small[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 p : small) {
    if (n == p) return true;
    if (n % p == 0) return false;
  }
  u64 d = n - 1;
  int s = 0;
  while (!(d & 1)) d >>= 1, ++s;
  for (u64 a : small) {
    u64 x = h_powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < s; ++i) {
      x = h_mulmod(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}
std::vector<u64> h_ntt_primes(int bits, u64 degree, size_t count, const std::vector<u64>& avoid) {
  const u64 step = 2 * degree, lo = 1ull << (bits - 1);
  u64 cand = (1ull << bits) - step + 1;
  std::vector<u64> out;
  while (out.size() < count && cand > lo) {
    if (h_is_prime(cand) && std::find(avoid.begin(), avoid.end(), cand) == avoid.end() &&
        std::find(out.begin(), out.end(), cand) == out.end())
      out.push_back(cand);
    cand -= step;
  }
  if (out.size() < count) fail(LCL_PARAMETER_ERROR, "prime search exhausted the requested bit range");
  return out;
}
u64 h_root_2n(u64 n, u64 q) {
  const u64 quot = (q - 1) / (2 * n);
  for (u64 g = 2; g < q; ++g) {
    const u64 r = h_powmod(g, quot, q);
    if (h_powmod(r, n, q) == q - 1) return r;
  }
  fail(LCL_PARAMETER_ERROR, "no primitive root found");
}
u64 h_shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
size_t h_brv(size_t x, int bits) {
  size_t r = 0;
  for (int i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
  return r;
}

// ------------------------------------------------------------ canonical embedding
// Host encode of a plaintext (ckks.cpp:263-307 with encoding.cpp:37-116),
// compiled without FP contraction so it reproduces the reference's default
// x86-64 build word for word. Used only for the 1/l plaintext of Multi-Krum
// averaging, which the reference also encodes on the host.
std::vector<long long> h_encode_rounded(const std::vector<double>& values, size_t degree,
                                        double scale) {
  const size_t h = degree / 2;
  const int logh = __builtin_ctzll(h);
  std::vector<double> br(h, 0.0), bi(h, 0.0);
  u64 g = 1;
  const u64 two_n = 2 * degree;
  for (size_t j = 0; j < values.size(); ++j) {
    br[(g - 1) / 4] = values[j];
    g = (g * 5) % two_n;
  }
  for (size_t i = 0; i < h; ++i) {
    const size_t r = h_brv(i, logh);
    if (i < r) {
      std::swap(br[i], br[r]);
      std::swap(bi[i], bi[r]);
    }
  }
  const double pi = 3.141592653589793238462643383279502884;
  for (size_t len = 2; len <= h; len <<= 1) {
    const size_t stride = h / len;
    for (size_t st = 0; st < h; st += len) {
      for (size_t k = 0; k < len / 2; ++k) {
        const double ang = 2.0 * pi * (double)(k * stride) / (double)h;
        const double wr = std::cos(ang), wi = -std::sin(ang);  // inverse: conj
        const size_t u = st + k, v = st + k + len / 2;
        const double xr = br[v], xi = bi[v];
        const double vr = xr * wr - xi * wi, vi = xr * wi + xi * wr;
        const double ur = br[u], ui = bi[u];
        br[u] = ur + vr;
        bi[u] = ui + vi;
        br[v] = ur - vr;
        bi[v] = ui - vi;
      }
    }
  }
  const double s = 1.0 / (double)h;
  for (size_t i = 0; i < h; ++i) {
    br[i] *= s;
    bi[i] *= s;
  }
  std::vector<long long> rounded(degree);
  for (size_t i = 0; i < h; ++i) {
    const double ang = pi * (double)i / (double)degree;
    const double tr = std::cos(ang), ti = -std::sin(ang);
    const double re = br[i] * tr - bi[i] * ti;
    const double im = br[i] * ti + bi[i] * tr;
    const double x0 = re * scale, x1 = im * scale;
    if (std::fabs(x0) >= 4.6e18 || std::fabs(x1) >= 4.6e18)
      fail(LCL_CAPACITY_ERROR, "scaled coefficient overflows 62 bits");
    rounded[i] = std::llround(x0);
    rounded[i + h] = std::llround(x1);
  }
  return rounded;
}

// ------------------------------------------------------------ device buffers
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  u64* get(size_t need_words) {
    const size_t need = need_words * 8;
    if (need > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      cuda_check(cudaMalloc(&p, need), "workspace alloc");
      bytes = need;
    }
    return static_cast<u64*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

RowMap make_map(const u64* base, u32 rpi, u64 row_stride, u64 item_stride, u32 ipg,
                u64 group_stride, const std::vector<u32>& primes) {
  RowMap m;
  std::memset(&m, 0, sizeof m);
  m.base = const_cast<u64*>(base);
  m.rows_per_item = rpi;
  m.row_stride = row_stride;
  m.item_stride = item_stride;
  m.items_per_group = ipg;
  m.group_stride = ipg == 1 ? item_stride : group_stride;
  for (u32 i = 0; i < rpi && i < 2 * LCL_MAXP; ++i) m.prime_of[i] = (unsigned char)primes[i];
  return m;
}

RowMap null_map() {
  RowMap m;
  std::memset(&m, 0, sizeof m);
  m.rows_per_item = 1;
  m.items_per_group = 1;
  return m;
}

}  // namespace

// ------------------------------------------------------------ context
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
  double bytes;  // algorithmic bytes moved by the launch
  double bfly;   // algorithmic radix-2 butterflies of the launch
};

struct lcl_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  size_t n = 0;
  int logn = 0;
  u32 full = 0;  // q primes; special at index full
  std::vector<u64> primes;
  double scale = 0;
  PrimeConst* d_primes = nullptr;
  ulonglong2* d_tw = nullptr;
  ulonglong2* d_itw = nullptr;
  double2* d_twf = nullptr;   // (w, w / q) doubles for FP64 rows
  double2* d_itwf = nullptr;
  // block-ordered copies for the 256-point block passes (ntt.cuh blk_tw_pos)
  ulonglong2* d_btw = nullptr;
  ulonglong2* d_bitw = nullptr;
  double2* d_btwf = nullptr;
  double2* d_bitwf = nullptr;
  u32 fp_mask = 0;            // primes whose rows run on the FP64 pipe
  bool pair_f64 = false;      // q-chain below 2^44: pair accumulation on the FP64 pipe
  u64* d_smod = nullptr;
  ulonglong2* d_pinv = nullptr;  // [(full+1) * (full+1)]: (q_div^-1 mod q_dst, shoup)
  u32* d_pairs = nullptr;
  size_t pairs_cap = 0;
  u32 pairs_n = 0;
  std::map<std::tuple<u32, u32, u32, u32>, uint2*> sched;  // pair_schedule cache
  u64* d_relin = nullptr;
  u64* d_relin_shoup = nullptr;
  std::map<size_t, u64*> d_rot;
  std::map<size_t, u64*> d_rot_shoup;
  std::map<size_t, u32*> d_perm;
  std::map<size_t, u32*> d_blkmap;  // two-pass rings: source block -> output block of the perm
  std::map<size_t, u32*> d_sigma;  // coefficient-domain automorphism (src | neg << 31)
  lcl_counts counts{};
  u64 launches = 0;
  bool prof_on = false;
  std::vector<ProfRec> prof;
  // workspace
  DevBuf ws_coef, ws_digits, ws_acc, ws_coefsp, ws_mid, ws_tern, ws_ctA, ws_ctB, ws_ctC, ws_pt,
      ws_c1inv;
  // Concurrent lanes: independent ciphertext groups of a batched key-switch
  // chain run on their own streams with their own workspaces, so the small,
  // latency-bound per-level kernels of one group fill the SMs the other
  // group's kernels leave idle (ramp-up, tails, memory stalls).
  struct Lane {
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    DevBuf ws_coef, ws_digits, ws_acc, ws_coefsp, ws_mid, ws_tern, ws_ctA, ws_ctB, ws_ctC, ws_c1inv;
  };
  std::vector<Lane> lanes;
  cudaEvent_t fork_ev = nullptr;
  bool in_lane = false;  // work is being enqueued on a lane: no nested lanes
  DevBuf ws_io_in, ws_io_sel, ws_io_dist, ws_io_agg, ws_dtern, ws_atern, ws_ptl, ws_enc, ws_enc_in;
  DevBuf ws_cal;   // calibrate()'s two rotated ciphertexts
  DevBuf ws_rows;  // DistanceMode::row_sums
  DevBuf ws_slots;  // KGC: decoded slots + entry values
  DevBuf ws_stage, ws_stage_sel, ws_err;  // LCLT blob staging + unpack error words: the unreduced pair ciphertexts
  // masked_aggregate's encode(1/l) plaintext, NTT'd on the device once per l
  size_t pt_l = 0;
  std::vector<u64> pt_host;
  // decode tables (Embedding, encoding.cpp:40-80), built on first decode
  double2* d_twist = nullptr;
  double2* d_roots = nullptr;
  u32* d_brv = nullptr;
  u32* d_slot = nullptr;
  DevBuf ws_dec;
  // overlapped host round: H2D / D2H copy streams and per-slice events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaStream_t unpk = nullptr;  // LCLT unpacking off the copy stream (host round)
  cudaStream_t d2h_agg = nullptr;  // the aggregate's D2H, independent of the pairs' copies
  cudaStream_t crit = nullptr;     // highest-priority streams for the host round's last two lanes
  cudaStream_t crit2 = nullptr;
  cudaStream_t lo = nullptr;       // lowest priority: the last group's slice accumulations
  cudaStream_t crit3 = nullptr;    // highest priority: the last group's aggregate slices
  std::vector<cudaEvent_t> unpk_ev;
  std::vector<cudaEvent_t> io_ev;

  u32 P() const { return full + 1; }
  u64 N() const { return (u64)n; }
  std::vector<u32> primes_0(u32 count) const {
    std::vector<u32> v(count);
    for (u32 i = 0; i < count; ++i) v[i] = i;
    return v;
  }
};

// Sampler (sampling.hpp:32-65, sampling.cpp): the reference's deterministic
// stream over std::mt19937_64 with its rejection-sampled bounded draws, so a
// client's encryptions consume exactly the reference's draws.
struct lcl_sampler {
  std::mt19937_64 engine;
  explicit lcl_sampler(u64 seed) : engine(seed) {}
  u64 raw() { return engine(); }
  u64 uniform_below(u64 bound) {  // sampling.cpp:34-41
    if ((bound & (bound - 1)) == 0) return raw() & (bound - 1);
    const u64 limit = ~u64{0} - (~u64{0} % bound) - 1;
    u64 x = raw();
    while (x > limit) x = raw();
    return x % bound;
  }
  double uniform_real() { return static_cast<double>(raw() >> 11) * 0x1.0p-53; }  // :43-45
  void ternary(size_t n, signed char* out) {  // :70-78
    for (size_t j = 0; j < n; ++j) out[j] = (signed char)((long)uniform_below(3) - 1);
  }
  void sparse_ternary(size_t n, size_t weight, signed char* out) {  // :80-98
    std::fill(out, out + n, 0);
    std::vector<size_t> idx(n);
    for (size_t i = 0; i < n; ++i) idx[i] = i;
    for (size_t i = 0; i < weight; ++i) {
      const size_t k = i + uniform_below(n - i);
      std::swap(idx[i], idx[k]);
      out[idx[i]] = uniform_below(2) == 0 ? 1 : -1;
    }
  }
  void cbd(size_t n, int eta, signed char* out) {  // :100-112
    const u64 mask = (eta == 32) ? ~u64{0} >> 32 : (u64{1} << eta) - 1;
    for (size_t j = 0; j < n; ++j) {
      const u64 bits = raw();
      out[j] = (signed char)(__builtin_popcountll(bits & mask) -
                             __builtin_popcountll((bits >> eta) & mask));
    }
  }
};

namespace {

void count_launch(lcl_context* c, u64 k = 1) { c->launches += k; }

NttTabs tabs(const lcl_context* c) {
  NttTabs t;
  t.tw = c->d_tw;
  t.itw = c->d_itw;
  t.twf = c->d_twf;
  t.itwf = c->d_itwf;
  t.btw = c->d_btw;
  t.bitw = c->d_bitw;
  t.btwf = c->d_btwf;
  t.bitwf = c->d_bitwf;
  t.primes = c->d_primes;
  t.fp_mask = c->fp_mask;
  t.logn = (u32)c->logn;
  return t;
}

// Field selection of a row map (ntt.cuh use_fp): 1 = every row's prime runs
// on the FP64 pipe, 2 = every row on the integer pipe, 0 = mixed.
int field_sel(const lcl_context* c, const RowMap& m) {
  bool fp = false, in = false;
  for (u32 r = 0; r < m.rows_per_item; ++r) ((c->fp_mask >> m.prime_of[r]) & 1u ? fp : in) = true;
  return fp && !in ? 1 : (in && !fp ? 2 : 0);
}
// Calls f(integral_constant<FS>) for the map's field selection.
template <class F>
void with_fs(int fs, F&& f) {
  if (fs == 1) f(std::integral_constant<int, 1>{});
  else if (fs == 2) f(std::integral_constant<int, 2>{});
  else f(std::integral_constant<int, 0>{});
}

void post_launch(lcl_context* c, u64 k = 1) {
  count_launch(c, k);
  cuda_check(cudaGetLastError(), "kernel launch");
}

// CUDA-event bracket around one launch when profiling is on (bench.py uses it
// to attribute the round's device time to kernels).
struct ProfScope {
  lcl_context* c;
  const char* name;
  double bytes;
  double bfly;
  cudaEvent_t a = nullptr;
  ProfScope(lcl_context* c_, const char* n, double b, double bf = 0)
      : c(c_), name(n), bytes(b), bfly(bf) {
    if (c->prof_on) {
      cudaEventCreate(&a);
      cudaEventRecord(a, c->stream);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b2;
      cudaEventCreate(&b2);
      cudaEventRecord(b2, c->stream);
      c->prof.push_back({name, a, b2, bytes, bfly});
    }
  }
};

// Algorithmic traffic of the functors (words per output row).
inline double load_rows(const PlainLoad&, double rows) { return rows; }
template <bool S>
inline double load_rows(const LiftLoadT<S>& l, double rows) { return rows / l.fan; }
inline double store_rows(const PlainStore&, double rows) { return rows; }
inline double store_rows(const DivRoundStore& s, double rows) {
  return rows * (2.0 + (s.add1.base ? 1.0 : 0.0)) + (s.add2.base ? rows / 2 : 0.0);
}
inline double store_rows(const DivRoundInvStore& s, double rows) {
  return store_rows(static_cast<const DivRoundStore&>(s), rows) + rows / 2;  // + the c1 inverse rows
}

// ------------------------------------------------------------ NTT launchers
RowMap mid_map(lcl_context* c, u32 rows, const RowMap& pm) {
  u64* mid = c->ws_mid.get((u64)rows * c->N());
  RowMap m = pm;
  m.base = mid;
  m.row_stride = c->N();
  m.item_stride = (u64)pm.rows_per_item * c->N();
  m.items_per_group = 1;
  m.group_stride = m.item_stride;
  return m;
}

template <class K>
void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
               "smem attribute");
}

template <int LOGN1, int E, class Loader, class Epi>
void fwd2(lcl_context* c, u32 rows, const RowMap& mid, const Loader& ld, const Epi& epi) {
  constexpr int N1 = 1 << LOGN1;
  constexpr size_t smem = (size_t)N1 * 16 * 8;
  static bool once = (allow_smem(ntt_col_fwd<LOGN1, E, Loader>, smem), true);
  (void)once;
  const u32 groups = (u32)(c->n >> LOGN1) >> 4;
  const double rb = 8.0 * c->N();
  const double bpr = 0.5 * c->N();  // butterflies per row per stage
  {
    ProfScope ps(c, std::is_same<Loader, PlainLoad>::value ? "ntt_col_fwd" : "ntt_col_fwd<lift>",
                 rb * (load_rows(ld, rows) + rows), bpr * rows * LOGN1);
    ntt_col_fwd<LOGN1, E, Loader><<<rows * groups, 16 * (N1 / E), smem, c->stream>>>(mid, ld, tabs(c));
  }
  {
    ProfScope ps(c, std::is_same<Epi, DivRoundStore>::value ? "ntt_blk_fwd<divround>" : "ntt_blk_fwd",
                 rb * (store_rows(epi, rows) + (std::is_same<Epi, PlainStore>::value ? rows : 0)),
                 bpr * rows * 8);
    constexpr int kMinB = std::is_same<Epi, DivRoundInvStore>::value ? LCL_INV_MINB : 16;
  with_fs(field_sel(c, mid), [&](auto FS) {
    ntt_blk_fwd<LOGN1, Epi, kMinB, decltype(FS)::value><<<rows * N1 / 4, 64, 0, c->stream>>>(mid, epi, tabs(c));
  });
  }
  post_launch(c, 2);
}

template <int LOGN1, int E, class Epi>
void inv2(lcl_context* c, u32 rows, const RowMap& in, const RowMap& mid, const Epi& epi) {
  constexpr int N1 = 1 << LOGN1;
  constexpr size_t smem = (size_t)N1 * 16 * 8;
  static bool once = (allow_smem(ntt_col_inv<LOGN1, E, Epi>, smem), true);
  (void)once;
  const u32 groups = (u32)(c->n >> LOGN1) >> 4;
  const double rb = 8.0 * c->N();
  const double bpr = 0.5 * c->N();
  {
    ProfScope ps(c, "ntt_blk_inv", rb * 2.0 * rows, bpr * rows * 8);
    with_fs(field_sel(c, in), [&](auto FS) {
      ntt_blk_inv<LOGN1, 1, decltype(FS)::value><<<rows * N1 / 4, 64, 0, c->stream>>>(in, mid, tabs(c));
    });
  }
  {
    ProfScope ps(c, "ntt_col_inv", rb * 2.0 * rows, bpr * rows * LOGN1);
    ntt_col_inv<LOGN1, E, Epi><<<rows * groups, 16 * (N1 / E), smem, c->stream>>>(mid, epi, tabs(c));
  }
  post_launch(c, 2);
}

// Forward NTT of `rows` rows whose prime layout is pm; the loader supplies
// coefficient-domain inputs and the epilogue consumes fully reduced outputs.
template <class Loader, class Epi>
void launch_fwd(lcl_context* c, u32 rows, const RowMap& pm, const Loader& ld, const Epi& epi) {
  if (rows == 0) return;
  if (c->logn <= 12) {
    ProfScope ps(c, "ntt_small_fwd", 8.0 * c->N() * (load_rows(ld, rows) + store_rows(epi, rows)),
                 0.5 * c->N() * rows * c->logn);
    ntt_small<false, Loader, Epi><<<rows, 256, c->n * 8, c->stream>>>(ld, epi, pm, tabs(c));
    post_launch(c);
    return;
  }
  const RowMap mid = mid_map(c, rows, pm);
  switch (c->logn) {
    case 13: fwd2<5, 16>(c, rows, mid, ld, epi); break;
    case 14: fwd2<6, 16>(c, rows, mid, ld, epi); break;
    case 15: fwd2<7, 16>(c, rows, mid, ld, epi); break;
    case 16: fwd2<8, 16>(c, rows, mid, ld, epi); break;
    case 17: fwd2<9, 32>(c, rows, mid, ld, epi); break;
    default: fail(LCL_PARAMETER_ERROR, "ring degree outside 2^3..2^17");
  }
}

// ---- split passes for the fused pipelines (two-pass rings only)
template <int LOGN1>
void blk_inv_n(lcl_context* c, u32 rows, const RowMap& in, const RowMap& out) {
  constexpr int N1 = 1 << LOGN1;
  ProfScope ps(c, "ntt_blk_inv", 16.0 * c->N() * rows, 0.5 * c->N() * rows * 8);
  with_fs(field_sel(c, in), [&](auto FS) {
    ntt_blk_inv<LOGN1, 1, decltype(FS)::value><<<rows * N1 / 4, 64, 0, c->stream>>>(in, out, tabs(c));
  });
}

template <int LOGN1, int E, int MINB>
void col_ilf_cfg(lcl_context* c, u32 src_rows, const RowMap& src, const RowMap& dst, u32 fan) {
  constexpr int N1 = 1 << LOGN1;
  constexpr size_t smem = (size_t)N1 * 16 * 8 * (LCL_COL_VSMEM && E == 16 ? 2 : 1);
  const u32 groups = (u32)(c->n >> LOGN1) >> 4;
  ProfScope ps(c, "ntt_col_inv_lift_fwd", 8.0 * c->N() * (src_rows + (double)src_rows * fan),
               0.5 * c->N() * LOGN1 * (src_rows + (double)src_rows * fan));
  // field-specialised instances for the key-switch shapes: ModUp (FP64
  // q-limb sources, mixed targets), ModDown (integer special-prime sources,
  // FP64 targets), rescale (FP64 -> FP64), all-integer (LCL_FP64=0)
  auto go = [&](auto FSS, auto FSD) {
    constexpr int A = decltype(FSS)::value, B = decltype(FSD)::value;
    static bool once = (allow_smem(ntt_col_inv_lift_fwd<LOGN1, E, MINB, A, B>, smem), true);
    (void)once;
    ntt_col_inv_lift_fwd<LOGN1, E, MINB, A, B><<<src_rows * groups, 16 * (N1 / E), smem, c->stream>>>(
        src, dst, fan, c->d_smod, c->P(), tabs(c));
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  const int fss = field_sel(c, src), fsd = field_sel(c, dst);
  if (fss == 1 && fsd == 0) go(I1{}, I0{});
  else if (fss == 2 && fsd == 1) go(I2{}, I1{});
  else if (fss == 1 && fsd == 1) go(I1{}, I1{});
  else if (fss == 2 && fsd == 2) go(I2{}, I2{});
  else go(I0{}, I0{});
}

// E = 16: 4 CTAs per SM (128 registers) -- measured cfg2 2.26 -> 1.95 ms,
// cfg3 24.3 -> 17.5 ms against the unconstrained build (252 registers,
// 3 CTAs); E = 32 (N = 2^17): 2 CTAs per SM (128 registers), rotate 46.1 ->
// 44.3 us per ciphertext. (E = 8 cannot work at N1 = 128: the two register
// phases need E^2 >= N1, i.e. R = N1 / E <= E.)
template <int LOGN1, int E>
void col_ilf_n(lcl_context* c, u32 src_rows, const RowMap& src, const RowMap& dst, u32 fan) {
  col_ilf_cfg<LOGN1, E, E == 16 ? LCL_COL_MINB : 2>(c, src_rows, src, dst, fan);
}

template <int LOGN1, class Epi>
void blk_fwd_n(lcl_context* c, u32 rows, const RowMap& mid, const Epi& epi) {
  constexpr int N1 = 1 << LOGN1;
  ProfScope ps(c,
               std::is_same<Epi, DivRoundStore>::value      ? "ntt_blk_fwd<divround>"
               : std::is_same<Epi, DivRoundInvStore>::value ? "ntt_blk_fwd<divround+inv>"
                                                            : "ntt_blk_fwd",
               8.0 * c->N() * (store_rows(epi, rows) + (std::is_same<Epi, PlainStore>::value ? rows : 0)),
               0.5 * c->N() * rows * (std::is_same<Epi, DivRoundInvStore>::value ? 12 : 8));
  // 16 CTAs per SM (64-register cap): measured cfg2 1.87 -> 1.49 ms, cfg3
  // 15.65 -> 11.44 ms against the unconstrained build (128 registers); the
  // same cap on ntt_blk_inv and a 10-CTA cap on modup_ip_blk were slower
  if constexpr (LCL_DR_TMA && (std::is_same<Epi, DivRoundStore>::value ||
                               std::is_same<Epi, DivRoundInvStore>::value)) {
    constexpr size_t smem = 4 * kDrGroupWords * 8;
    static bool once = (allow_smem(ntt_blk_fwd_dr_tma<LOGN1, Epi, LCL_DR_MINB>, smem), true);
    (void)once;
    ntt_blk_fwd_dr_tma<LOGN1, Epi, LCL_DR_MINB><<<rows * N1 / 4, 64, smem, c->stream>>>(mid, epi, tabs(c));
  } else {
    constexpr int kMinB = std::is_same<Epi, DivRoundInvStore>::value ? LCL_INV_MINB : 16;
    with_fs(field_sel(c, mid), [&](auto FS) {
      ntt_blk_fwd<LOGN1, Epi, kMinB, decltype(FS)::value><<<rows * N1 / 4, 64, 0, c->stream>>>(mid, epi,
                                                                                             tabs(c));
    });
  }
}

// Calls f(LOGN1, E) with compile-time constants for the two-pass ring sizes.
template <class F>
void dispatch_logn(lcl_context* c, F&& f) {
  switch (c->logn) {
    case 13: f(std::integral_constant<int, 5>{}, std::integral_constant<int, 16>{}); break;
    case 14: f(std::integral_constant<int, 6>{}, std::integral_constant<int, 16>{}); break;
    case 15: f(std::integral_constant<int, 7>{}, std::integral_constant<int, 16>{}); break;
    case 16: f(std::integral_constant<int, 8>{}, std::integral_constant<int, 16>{}); break;
    case 17: f(std::integral_constant<int, 9>{}, std::integral_constant<int, 32>{}); break;
    default: fail(LCL_PARAMETER_ERROR, "ring degree outside 2^13..2^17");
  }
}

// Inverse NTT of `src_rows` rows (map `in`) fused with the centred lift into
// `fan` destination rows each and their forward column pass; the output
// (dst map) is ready for a forward block pass. Returns nothing; two launches.
void inv_lift_fwd_cols(lcl_context* c, u32 src_rows, const RowMap& in, const RowMap& dst,
                       u32 fan) {
  const u64 N = c->N();
  u64* tmp = c->ws_coef.get((u64)src_rows * N);
  RowMap t = in;
  t.base = tmp;
  t.row_stride = N;
  t.item_stride = (u64)in.rows_per_item * N;
  t.items_per_group = 1;
  t.group_stride = t.item_stride;
  dispatch_logn(c, [&](auto L1, auto E) {
    blk_inv_n<decltype(L1)::value>(c, src_rows, in, t);
    col_ilf_n<decltype(L1)::value, decltype(E)::value>(c, src_rows, t, dst, fan);
  });
  post_launch(c, 2);
}

// Same, for source rows whose inverse block pass already ran.
void lift_fwd_cols_preinv(lcl_context* c, u32 src_rows, const RowMap& src_inv, const RowMap& dst,
                          u32 fan) {
  dispatch_logn(c, [&](auto L1, auto E) {
    col_ilf_n<decltype(L1)::value, decltype(E)::value>(c, src_rows, src_inv, dst, fan);
  });
  post_launch(c);
}

template <class Epi>
void blk_fwd_only(lcl_context* c, u32 rows, const RowMap& mid, const Epi& epi) {
  dispatch_logn(c, [&](auto L1, auto) { blk_fwd_n<decltype(L1)::value>(c, rows, mid, epi); });
  post_launch(c);
}

LiftLoad lift_from(lcl_context* c, const RowMap& src, u32 rows_per_item, u32 fan) {
  LiftLoad l;
  l.src = src;
  l.rows_per_item = rows_per_item;
  l.fan = fan;
  l.nprimes = c->P();
  l.primes = c->d_primes;
  l.smod = c->d_smod;
  l.sigma = nullptr;
  return l;
}

template <int LOGN1, int M>
void modup_ip_launch(lcl_context* c, u32 B, const u64* mid, const u64* c1, u64 c1_stride,
                     const u32* perm, const u64* key, const u64* key_aux, u64* acc) {
  constexpr int N1 = 1 << LOGN1;
  const double rb = 8.0 * c->N();
  ProfScope ps(c, perm ? "modup_ip_blk<perm>" : "modup_ip_blk",
               rb * ((double)B * M * M + B * M + 4.0 * M * (M + 1) + 2.0 * B * (M + 1)),
               0.5 * c->N() * B * M * M * 8);
  constexpr size_t smem = modup_smem_bytes(LCL_MODUP_G);
  const u32 bq = (B + LCL_MODUP_G - 1) / LCL_MODUP_G;
  const bool sp_int = !((c->fp_mask >> c->full) & 1u);
  const bool q_fp = (c->fp_mask & ((1u << M) - 1)) == ((1u << M) - 1);
  if (LCL_MODUP_SPLIT && sp_int && q_fp) {
    // the special target (integer field) then the M q targets (FP64 field)
    static bool once = (allow_smem(modup_ip_blk<LOGN1, M, 2>, smem), allow_smem(modup_ip_blk<LOGN1, M, 1>, smem),
                        true);
    (void)once;
    modup_ip_blk<LOGN1, M, 2><<<bq * N1, 16 * LCL_MODUP_G, smem, c->stream>>>(
        B, mid, c1, c1_stride, perm, key, key_aux, c->full, acc, tabs(c), 0);
    modup_ip_blk<LOGN1, M, 1><<<bq * M * N1, 16 * LCL_MODUP_G, smem, c->stream>>>(
        B, mid, c1, c1_stride, perm, key, key_aux, c->full, acc, tabs(c), 1);
    count_launch(c);
    return;
  }
  static bool once = (allow_smem(modup_ip_blk<LOGN1, M, 0>, smem), true);
  (void)once;
  modup_ip_blk<LOGN1, M, 0><<<bq * (M + 1) * N1, 16 * LCL_MODUP_G, smem, c->stream>>>(
      B, mid, c1, c1_stride, perm, key, key_aux, c->full, acc, tabs(c), 0);
}

template <int LOGN1>
void modup_ip_n(lcl_context* c, u32 B, u32 m, const u64* mid, const u64* c1, u64 c1_stride,
                const u32* perm, const u64* key, const u64* key_shoup, u64* acc) {
  switch (m) {
    case 1: modup_ip_launch<LOGN1, 1>(c, B, mid, c1, c1_stride, perm, key, key_shoup, acc); break;
    case 2: modup_ip_launch<LOGN1, 2>(c, B, mid, c1, c1_stride, perm, key, key_shoup, acc); break;
    case 3: modup_ip_launch<LOGN1, 3>(c, B, mid, c1, c1_stride, perm, key, key_shoup, acc); break;
    case 4: modup_ip_launch<LOGN1, 4>(c, B, mid, c1, c1_stride, perm, key, key_shoup, acc); break;
    case 5: modup_ip_launch<LOGN1, 5>(c, B, mid, c1, c1_stride, perm, key, key_shoup, acc); break;
    case 6: modup_ip_launch<LOGN1, 6>(c, B, mid, c1, c1_stride, perm, key, key_shoup, acc); break;
    default: fail(LCL_PARAMETER_ERROR, "fused key switching supports up to 6 live limbs");
  }
  post_launch(c);
}

template <class Epi>
void launch_inv(lcl_context* c, u32 rows, const RowMap& in, const Epi& epi) {
  if (rows == 0) return;
  if (c->logn <= 12) {
    ProfScope ps(c, "ntt_small_inv", 8.0 * c->N() * 2.0 * rows, 0.5 * c->N() * rows * c->logn);
    ntt_small<true, PlainLoad, Epi><<<rows, 256, c->n * 8, c->stream>>>(PlainLoad{in}, epi, in,
                                                                       tabs(c));
    post_launch(c);
    return;
  }
  const RowMap mid = mid_map(c, rows, in);
  switch (c->logn) {
    case 13: inv2<5, 16>(c, rows, in, mid, epi); break;
    case 14: inv2<6, 16>(c, rows, in, mid, epi); break;
    case 15: inv2<7, 16>(c, rows, in, mid, epi); break;
    case 16: inv2<8, 16>(c, rows, in, mid, epi); break;
    case 17: inv2<9, 32>(c, rows, in, mid, epi); break;
    default: fail(LCL_PARAMETER_ERROR, "ring degree outside 2^3..2^17");
  }
}


// ------------------------------------------------------------ key switching
// decompose_for_keyswitch (ckks.cpp:464-481): the c1 / d2 rows of B items
// (map `in`, rows_per_item = m) -> digits [B][m][m+1][N] in HBM.
u64* ks_decompose(lcl_context* c, const RowMap& in, u32 B, u32 m, const u32* sigma = nullptr) {
  const u64 N = c->N();
  u64* coef = c->ws_coef.get((u64)B * m * N);
  const RowMap coef_map = make_map(coef, m, N, m * N, 1, 0, c->primes_0(m));
  launch_inv(c, B * m, in, PlainStore{coef_map});
  u64* dig = c->ws_digits.get((u64)B * m * (m + 1) * N);
  std::vector<u32> dp(m * (m + 1));
  for (u32 j = 0; j < m; ++j)
    for (u32 t = 0; t <= m; ++t) dp[j * (m + 1) + t] = t < m ? t : c->full;
  const RowMap dig_map = make_map(dig, m * (m + 1), N, (u64)m * (m + 1) * N, 1, 0, dp);
  if (sigma) {
    const LiftLoad base = lift_from(c, coef_map, m * (m + 1), m + 1);
    LiftSigmaLoad lift;
    std::memcpy(&lift, &base, sizeof base);
    lift.sigma = sigma;
    launch_fwd(c, B * m * (m + 1), dig_map, lift, PlainStore{dig_map});
  } else {
    launch_fwd(c, B * m * (m + 1), dig_map, lift_from(c, coef_map, m * (m + 1), m + 1),
               PlainStore{dig_map});
  }
  return dig;
}

u64* ks_ip(lcl_context* c, const u64* dig, u32 B, u32 m, const u64* key, const u32* perm) {
  const u64 N = c->N();
  u64* acc = c->ws_acc.get((u64)B * 2 * (m + 1) * N);
  constexpr u32 IB = 8;
  const dim3 grid((u32)(((u64)(m + 1) * N + 255) / 256), (B + IB - 1) / IB);
  ProfScope ps(c, perm ? "ks_inner_product<perm>" : "ks_inner_product",
               8.0 * N * ((double)B * m * (m + 1) + 2.0 * m * (m + 1) + 2.0 * B * (m + 1)));
#define LCL_IP(MM)                                                                           \
  case MM:                                                                                   \
    lcl::ks_inner_product<MM, IB><<<grid, 256, 0, c->stream>>>(dig, B, key, c->full, perm, acc, \
                                                               c->logn, c->d_primes);        \
    break;
  switch (m) {
    LCL_IP(1) LCL_IP(2) LCL_IP(3) LCL_IP(4) LCL_IP(5) LCL_IP(6) LCL_IP(7) LCL_IP(8)
    default: fail(LCL_PARAMETER_ERROR, "key switching supports up to 8 live limbs");
  }
#undef LCL_IP
  post_launch(c);
  return acc;
}

// One modup_ip_hoist launch: the ModUp block pass of the digits in mid
// (column-pass output, [B][m][m][N]) feeding the inner products of ns steps
// into acc + s * acc_step ([B][2][m+1][N] each).
void hoist_launch(lcl_context* c, u32 B, u32 m, const u64* mid, const u64* c1, u64 c1_stride,
                  const HoistSteps& hs, u32 ns, u64* acc, u64 acc_step) {
  const double rb = 8.0 * c->N();
  {
    ProfScope ps(c, ns == 1 ? "modup_ip_hoist<1>" : "modup_ip_hoist",
                 rb * ((double)B * m * m + (double)B * m + 2.0 * ns * m * (m + 1) + 2.0 * ns * B * (m + 1)),
                 0.5 * c->N() * B * m * m * 8);
    dispatch_logn(c, [&](auto L1, auto) {
      constexpr int LOGN1 = decltype(L1)::value;
      const u32 grid = ((B + 3) / 4) * (m + 1) * (1u << LOGN1);
#define LCL_HOIST(MM)                                                                        \
  case MM:                                                                                   \
    modup_ip_hoist<LOGN1, MM><<<grid, 64, 0, c->stream>>>(B, mid, c1, c1_stride, hs, ns,      \
                                                          c->full, acc, acc_step, tabs(c));  \
    break;
      switch (m) {
        LCL_HOIST(1) LCL_HOIST(2) LCL_HOIST(3) LCL_HOIST(4)
        default: fail(LCL_PARAMETER_ERROR, "hoisted key switching supports up to 4 live limbs");
      }
#undef LCL_HOIST
    });
  }
  post_launch(c);
}

// decompose_for_keyswitch + inner product (ckks.cpp:464-518) for the c1 / d2
// limbs of B items: `in` maps them (rows_per_item = m); c1 / c1_stride address
// the same limbs for the identity digits. sigma / perm: the rotation's
// coefficient- / evaluation-domain automorphism (nullptr for relinearize).
// Returns acc [B][2][m+1][N].
bool ks_fused(const lcl_context* c, u32 m) { return c->logn >= 13 && m <= 6; }

// preinv: the c1 limbs' inverse block pass already ran (fused into the
// previous level's divide-and-round, rows [B][m][N]); fused path only.
u64* ks_switch(lcl_context* c, const RowMap& in, const u64* c1, u64 c1_stride, u32 B, u32 m,
               const u32* sigma, const u32* perm, const u64* key, const u64* key_shoup,
               const u64* preinv = nullptr, const u32* blkmap = nullptr) {
  if (!ks_fused(c, m)) {
    u64* dig = ks_decompose(c, in, B, m, sigma);
    return ks_ip(c, dig, B, m, key, nullptr);
  }
  const u64 N = c->N();
  // inverse NTT of the m limbs fused with the lift into the m non-identity
  // targets of each digit (b, j, t'), t = t' < j ? t' : t' + 1
  u64* mid = c->ws_digits.get((u64)B * m * m * N);
  std::vector<u32> dp(m * m);
  for (u32 j = 0; j < m; ++j)
    for (u32 tp = 0; tp < m; ++tp) {
      const u32 t = tp < j ? tp : tp + 1;
      dp[j * m + tp] = t < m ? t : c->full;
    }
  const RowMap mid_map = make_map(mid, m * m, N, (u64)m * m * N, 1, 0, dp);
  if (preinv)
    lift_fwd_cols_preinv(c, B * m, make_map(preinv, m, N, (u64)m * N, 1, 0, c->primes_0(m)),
                         mid_map, m);
  else
    inv_lift_fwd_cols(c, B * m, in, mid_map, m);
  u64* acc = c->ws_acc.get((u64)B * 2 * (m + 1) * N);
  if (LCL_ROT_HOIST && perm && blkmap && m <= 4) {
    // a single rotation through the hoisted kernel (digits parked in shared
    // memory, the inner product from them with register accumulators)
    HoistSteps hs{};
    hs.perm[0] = perm;
    hs.blkmap[0] = blkmap;
    hs.key[0] = key;
    hs.key_aux[0] = key_shoup;
    hoist_launch(c, B, m, mid, c1, c1_stride, hs, 1, acc, (u64)B * 2 * (m + 1) * N);
    return acc;
  }
  // (Running the special rows' inverse block stages inside modup_ip_blk was
  // measured slower on cfg2, 8.91 vs 8.77 ms: it lengthens the special-target
  // CTAs by as much as the standalone ntt_blk_inv costs.)
  dispatch_logn(c, [&](auto L1, auto) {
    modup_ip_n<decltype(L1)::value>(c, B, m, mid, c1, c1_stride, perm, key, key_shoup, acc);
  });
  (void)sigma;  // two-pass rings permute block-locally inside modup_ip_blk
  return acc;
}

// Hoisted key switches (hoisted_rotations, ckks.cpp:582-612) of the c1 limbs
// of B items (map `in`; c1 / c1_stride address the same limbs) for every
// rotation step of `steps`: the ModUp inverse NTT + lift + column pass runs
// once, then one modup_ip_hoist launch per group of <= kHoistMax steps
// transforms the digits' blocks once and forms every step's inner product;
// each(step index, acc [B][2][m+1][N]) then runs that step's ModDown.
// Rings below 2^13 or more than 4 live limbs use the materialised digits.
const u64* rot_key(lcl_context* c, size_t step);

template <class Each>
void ks_hoisted(lcl_context* c, const RowMap& in, const u64* c1, u64 c1_stride, u32 B, u32 m,
                const std::vector<size_t>& steps, Each&& each) {
  const u64 N = c->N();
  if (c->logn < 13 || m > 4) {
    u64* dig = ks_decompose(c, in, B, m);
    for (size_t s = 0; s < steps.size(); ++s)
      each(s, ks_ip(c, dig, B, m, rot_key(c, steps[s]), c->d_perm.at(steps[s])));
    return;
  }
  u64* mid = c->ws_digits.get((u64)B * m * m * N);
  std::vector<u32> dp(m * m);
  for (u32 j = 0; j < m; ++j)
    for (u32 tp = 0; tp < m; ++tp) {
      const u32 t = tp < j ? tp : tp + 1;
      dp[j * m + tp] = t < m ? t : c->full;
    }
  inv_lift_fwd_cols(c, B * m, in, make_map(mid, m * m, N, (u64)m * m * N, 1, 0, dp), m);
  const u64 acc_step = (u64)B * 2 * (m + 1) * N;
  const size_t G = std::min<size_t>(steps.size(), kHoistMax);
  u64* acc = c->ws_acc.get(G * acc_step);
  for (size_t s0 = 0; s0 < steps.size(); s0 += kHoistMax) {
    const u32 ns = (u32)std::min<size_t>(kHoistMax, steps.size() - s0);
    HoistSteps hs{};
    for (u32 i = 0; i < ns; ++i) {
      const size_t st = steps[s0 + i];
      hs.perm[i] = c->d_perm.at(st);
      hs.blkmap[i] = c->d_blkmap.at(st);
      hs.key[i] = rot_key(c, st);
      hs.key_aux[i] = c->d_rot_shoup.at(st);
    }
    hoist_launch(c, B, m, mid, c1, c1_stride, hs, ns, acc, acc_step);
    for (u32 i = 0; i < ns; ++i) each(s0 + i, acc + i * acc_step);
  }
}

// ModDown of acc [B][2][m+1][N] into `out` (items (b, x), rows_per_item m,
// 2 items per group) with the fused output additions; c1inv: also leave the
// next key switch's inverse block pass over out's c1 limbs there.
void ks_moddown(lcl_context* c, const u64* acc, u32 B, u32 m, const RowMap& out,
                const RowMap& add1, const RowMap& add2, const u32* perm,
                u64* c1inv = nullptr) {
  const u64 N = c->N();
  const RowMap sp_in = make_map(acc + (u64)m * N, 1, N, (m + 1) * N, 1, 0, {c->full});
  DivRoundStore epi;
  epi.out = out;
  epi.x = make_map(acc, m, N, (m + 1) * N, 1, 0, c->primes_0(m));
  epi.add1 = add1;
  epi.add2 = add2;
  epi.perm = perm;
  epi.pinv = c->d_pinv + (u64)c->full * c->P();
  if (c->logn >= 13) {
    // inverse NTT of the special rows + lift into the m q-primes + forward
    // column pass fused, then the block pass with the divide-and-round epilogue
    u64* mid = c->ws_mid.get((u64)B * 2 * m * N);
    const RowMap mid_map = make_map(mid, m, N, (u64)m * N, 1, 0, c->primes_0(m));
    inv_lift_fwd_cols(c, 2 * B, sp_in, mid_map, m);
    if (c1inv) {
      // also the next key switch's inverse block pass over the c1 limbs
      DivRoundInvStore ie;
      static_cast<DivRoundStore&>(ie) = epi;
      ie.inv_out = make_map(c1inv, m, N, 0, 2, (u64)m * N, c->primes_0(m));
      blk_fwd_only(c, 2 * B * m, mid_map, ie);
    } else {
      blk_fwd_only(c, 2 * B * m, mid_map, epi);
    }
    return;
  }
  need(!c1inv, LCL_USAGE_ERROR, "fused next-level inverse needs a two-pass ring");
  u64* csp = c->ws_coefsp.get((u64)B * 2 * N);
  const RowMap sp_map = make_map(csp, 1, N, N, 1, 0, {c->full});
  launch_inv(c, 2 * B, sp_in, PlainStore{sp_map});
  launch_fwd(c, 2 * B * m, out, lift_from(c, sp_map, m, m), epi);
}

RowMap ct_map(const u64* base, u32 m, u64 N, u64 ct_stride) {
  std::vector<u32> p(m);
  for (u32 i = 0; i < m; ++i) p[i] = i;
  return make_map(base, m, N, (u64)m * N, 2, ct_stride, p);
}

// relinearize (ckks.cpp:522-534) over a batch of ternaries [B][3][m][N].
void relinearize_batch(lcl_context* c, const u64* tern, u32 B, u32 m, u64* out) {
  if (!c->d_relin) fail(LCL_KEY_ERROR, "no relinearization key uploaded");
  const u64 N = c->N();
  const RowMap d2 = make_map(tern + 2ull * m * N, m, N, 3ull * m * N, 1, 0, c->primes_0(m));
  u64* acc = ks_switch(c, d2, tern + 2ull * m * N, 3ull * m * N, B, m, nullptr, nullptr,
                       c->d_relin, c->d_relin_shoup);
  ks_moddown(c, acc, B, m, ct_map(out, m, N, 2ull * m * N), ct_map(tern, m, N, 3ull * m * N),
             null_map(), nullptr);
  c->counts.relinearizations += B;
  c->counts.mod_ups += B;
}

// rescale (ckks.cpp:536-547): [B][2][m] -> [B][2][m-1] (in and out may not alias).
void rescale_batch(lcl_context* c, const u64* ct, u32 B, u32 m, u64* out) {
  if (m < 2) fail(LCL_DEPTH_EXHAUSTED, "no prime left to rescale by");
  const u64 N = c->N();
  const RowMap last_in = make_map(ct + (u64)(m - 1) * N, 1, N, (u64)m * N, 2, 2ull * m * N, {m - 1});
  DivRoundStore epi;
  epi.out = ct_map(out, m - 1, N, 2ull * (m - 1) * N);
  epi.x = ct_map(ct, m - 1, N, 2ull * m * N);
  epi.x.item_stride = (u64)m * N;
  epi.add1 = null_map();
  epi.add2 = null_map();
  epi.perm = nullptr;
  epi.pinv = c->d_pinv + (u64)(m - 1) * c->P();
  if (c->logn >= 13) {
    u64* mid = c->ws_mid.get((u64)B * 2 * (m - 1) * N);
    const RowMap mid_map = make_map(mid, m - 1, N, (u64)(m - 1) * N, 1, 0, c->primes_0(m - 1));
    inv_lift_fwd_cols(c, 2 * B, last_in, mid_map, m - 1);
    blk_fwd_only(c, 2 * B * (m - 1), mid_map, epi);
  } else {
    u64* last = c->ws_coefsp.get((u64)B * 2 * N);
    const RowMap last_map = make_map(last, 1, N, N, 1, 0, {m - 1});
    launch_inv(c, 2 * B, last_in, PlainStore{last_map});
    launch_fwd(c, 2 * B * (m - 1), epi.out, lift_from(c, last_map, m - 1, m - 1), epi);
  }
  c->counts.rescales += B;
}

const u64* rot_key(lcl_context* c, size_t step) {
  auto it = c->d_rot.find(step);
  if (it == c->d_rot.end()) fail(LCL_KEY_ERROR, "no rotation key for the requested step");
  return it->second;
}

// out = in + rotate(in, step) over B ciphertexts (one slot_reduce level,
// distance.cpp:235-237), or plain rotate when accumulate == false.
// preinv_in: in's c1 inverse block pass (from the previous level), or null;
// preinv_out: where to leave out's (fused into this level's divide-and-round).
void rotate_level(lcl_context* c, const u64* in, u32 B, u32 m, size_t step, u64* out,
                  bool accumulate, const u64* preinv_in = nullptr, u64* preinv_out = nullptr) {
  const u64 N = c->N();
  const u64* key = rot_key(c, step);
  const u32* perm = c->d_perm.at(step);
  const RowMap c1 = make_map(in + (u64)m * N, m, N, 2ull * m * N, 1, 0, c->primes_0(m));
  // two-pass rings: the Galois permutation is applied block-locally inside the
  // fused ModUp + inner-product pass; small rings lift through the
  // coefficient-domain automorphism instead.
  const u32* sigma = c->logn < 13 ? c->d_sigma.at(step) : nullptr;
  u64* acc = ks_switch(c, c1, in + (u64)m * N, 2ull * m * N, B, m, sigma, perm, key,
                       c->d_rot_shoup.at(step), preinv_in,
                       c->logn >= 13 ? c->d_blkmap.at(step) : nullptr);
  const RowMap inm = ct_map(in, m, N, 2ull * m * N);
  ks_moddown(c, acc, B, m, ct_map(out, m, N, 2ull * m * N), accumulate ? inm : null_map(), inm,
             perm, preinv_out);
  c->counts.rotations += B;
  c->counts.mod_ups += B;
  if (accumulate) c->counts.additions += B;
}

size_t norm_step(lcl_context* c, size_t step) { return step % (c->n / 2); }

// Swaps the context's stream and key-switch workspaces with lane g's.
void swap_lane(lcl_context* c, u32 g) {
  auto& ln = c->lanes[g];
  std::swap(c->stream, ln.stream);
  std::swap(c->ws_coef, ln.ws_coef);
  std::swap(c->ws_digits, ln.ws_digits);
  std::swap(c->ws_acc, ln.ws_acc);
  std::swap(c->ws_coefsp, ln.ws_coefsp);
  std::swap(c->ws_mid, ln.ws_mid);
  std::swap(c->ws_tern, ln.ws_tern);
  std::swap(c->ws_ctA, ln.ws_ctA);
  std::swap(c->ws_ctB, ln.ws_ctB);
  std::swap(c->ws_ctC, ln.ws_ctC);
  std::swap(c->ws_c1inv, ln.ws_c1inv);
}

// Two lanes pay off when a level's working set is L2-sized (cfg2: 45 x 3
// limbs x 2^15, 7.27 -> 7.07 ms); at cfg3 (190 x 3 x 2^16) the kernels
// already fill the SMs and a second lane only adds contention (92.8 -> 95.9).
u32 lane_count(lcl_context* c, u32 B, u32 m) {
  static const int env = [] {
    const char* e = std::getenv("LCL_LANES");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  if (c->prof_on || c->in_lane) return 1;  // serial attribution / no nesting
  const u32 want = env ? (u32)env : ((u64)B * m * c->N() <= (8ull << 20) ? 2u : 1u);
  return std::min<u32>(want, std::max<u32>(1, B / 8));
}

void ensure_lanes(lcl_context* c, u32 G) {
  while (c->lanes.size() < G) {
    c->lanes.emplace_back();
    auto& ln = c->lanes.back();
    cuda_check(cudaStreamCreateWithFlags(&ln.stream, cudaStreamNonBlocking), "lane stream");
    cuda_check(cudaEventCreateWithFlags(&ln.done, cudaEventDisableTiming), "lane event");
  }
  if (!c->fork_ev) cuda_check(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming), "fork event");
}

// Runs f() with the context's stream and key-switch workspaces swapped for
// lane g's (no nested lanes inside).
template <class F>
void on_lane(lcl_context* c, u32 g, F&& f) {
  swap_lane(c, g);
  c->in_lane = true;
  try {
    f();
  } catch (...) {
    c->in_lane = false;
    swap_lane(c, g);
    throw;
  }
  c->in_lane = false;
  swap_lane(c, g);
}

// Runs f(first, count) for G contiguous groups of [0, B) concurrently, group g
// on lane g (fork / join through events on the context stream, so the lanes
// are captured into the same CUDA graph as the rest of the round).
template <class F>
void run_lanes(lcl_context* c, u32 B, u32 G, F&& f) {
  if (G <= 1) {
    f(0u, B);
    return;
  }
  ensure_lanes(c, G);
  cuda_check(cudaEventRecord(c->fork_ev, c->stream), "fork");
  for (u32 g = 0; g < G; ++g) {
    const u32 b0 = (u32)((u64)B * g / G), b1 = (u32)((u64)B * (g + 1) / G);
    cuda_check(cudaStreamWaitEvent(c->lanes[g].stream, c->fork_ev, 0), "lane wait");
    swap_lane(c, g);
    try {
      f(b0, b1 - b0);
    } catch (...) {
      swap_lane(c, g);
      throw;
    }
    swap_lane(c, g);
    cuda_check(cudaEventRecord(c->lanes[g].done, c->lanes[g].stream), "lane done");
  }
  for (u32 g = 0; g < G; ++g)
    cuda_check(cudaStreamWaitEvent(c->stream, c->lanes[g].done, 0), "join");
}

void slot_reduce_serial(lcl_context* c, const u64* in, u32 B, u32 m, size_t width, size_t k,
                        u64* out);

// slot_reduce (distance.cpp:214-240) over B ciphertexts; in and out may alias.
// The B chains are independent: they run as concurrent lanes.
void slot_reduce_batch(lcl_context* c, const u64* in, u32 B, u32 m, size_t width, size_t k,
                       u64* out) {
  const u64 words = 2ull * m * c->N();
  run_lanes(c, B, lane_count(c, B, m), [&](u32 b0, u32 nb) {
    slot_reduce_serial(c, in + b0 * words, nb, m, width, k, out + b0 * words);
  });
}

void slot_reduce_serial(lcl_context* c, const u64* in, u32 B, u32 m, size_t width, size_t k,
                        u64* out) {
  if (width == 0 || (width & (width - 1))) fail(LCL_WIDTH_ERROR, "reduction width must be a power of two");
  if (width > c->n / 2) fail(LCL_WIDTH_ERROR, "reduction width exceeds the slot count");
  if (k == 0) fail(LCL_PARAMETER_ERROR, "unfold factor starts at 1");
  const u64 N = c->N();
  const u64 words = (u64)B * 2 * m * N;
  if (width == 1) {
    if (out != in) cudaMemcpyAsync(out, in, words * 8, cudaMemcpyDeviceToDevice, c->stream);
    return;
  }
  const size_t levels = __builtin_ctzll(width);
  const size_t unf = std::min(k - 1, levels);
  // validate keys up front (the reference raises KeyError before any work
  // lands in the output for the first missing step)
  for (size_t u = 1; unf >= 1 && u < (size_t{1} << unf); ++u) rot_key(c, norm_step(c, u));
  for (size_t j = unf; j < levels; ++j) rot_key(c, norm_step(c, size_t{1} << j));
  u64* bufs[2] = {c->ws_ctB.get(words), c->ws_ctC.get(words)};
  int cur = -1;  // -1: current value lives in `in`
  auto cur_ptr = [&]() -> const u64* { return cur < 0 ? in : bufs[cur]; };
  if (unf >= 1) {
    // hoisted batch: one decomposition of in.c1, every step reuses it.
    const RowMap c1 = make_map(in + (u64)m * N, m, N, 2ull * m * N, 1, 0, c->primes_0(m));
    c->counts.mod_ups += B;
    const RowMap base = ct_map(in, m, N, 2ull * m * N);
    std::vector<size_t> hsteps;
    for (size_t u = 1; u < (size_t{1} << unf); ++u) hsteps.push_back(norm_step(c, u));
    ks_hoisted(c, c1, in + (u64)m * N, 2ull * m * N, B, m, hsteps, [&](size_t i, u64* acc) {
      const int nxt = cur < 0 ? 0 : 1 - cur;
      ks_moddown(c, acc, B, m, ct_map(bufs[nxt], m, N, 2ull * m * N),
                 ct_map(cur_ptr(), m, N, 2ull * m * N), base, c->d_perm.at(hsteps[i]));
      cur = nxt;
      c->counts.rotations += B;
      c->counts.additions += B;
    });
  }
  // each level leaves its output's c1 inverse block pass for the next one
  // (two-pass rings); one buffer suffices: a level's column pass has read it
  // before the same level's divide-and-round rewrites it
  const bool chain = ks_fused(c, m);
  u64* pre = chain ? c->ws_c1inv.get((u64)B * m * N) : nullptr;
  for (size_t j = unf; j < levels; ++j) {
    const int nxt = cur < 0 ? 0 : 1 - cur;
    rotate_level(c, cur_ptr(), B, m, norm_step(c, size_t{1} << j), bufs[nxt], true,
                 chain && j > unf ? pre : nullptr, chain && j + 1 < levels ? pre : nullptr);
    cur = nxt;
  }
  cudaMemcpyAsync(out, cur_ptr(), words * 8, cudaMemcpyDeviceToDevice, c->stream);
}

void ensure_pairs(lcl_context* c, u32 n) {
  if (c->pairs_n == n) return;
  const size_t np = (size_t)n * (n - 1) / 2;
  std::vector<u32> h;
  h.reserve(np);
  for (u32 i = 0; i < n; ++i)
    for (u32 j = i + 1; j < n; ++j) h.push_back(i | (j << 16));
  if (np > c->pairs_cap) {
    if (c->d_pairs) cudaFree(c->d_pairs);
    cuda_check(cudaMalloc(&c->d_pairs, np * 4), "pairs alloc");
    c->pairs_cap = np;
  }
  cuda_check(cudaMemcpy(c->d_pairs, h.data(), np * 4, cudaMemcpyHostToDevice), "pairs upload");
  c->pairs_n = n;
}

// Lazy ternary accumulators for pairs [p0, p1) over chunks [c0, c1). Tiles of
// TE slots, TE / EPT threads per pair, up to 256 pairs per CTA: each client
// word is read from HBM once per pair group. STAGES chunks are in flight per
// CTA (one CTA per SM: the accumulators of 190 pairs x 8 slots fill the
// register file, so the copy pipeline, not occupancy, hides HBM latency).
template <int TE, int EPT, int STAGES>
void pair_accumulate_cfg(lcl_context* c, const u64* clients, u32 n, u32 chunks, u32 c0,
                         u32 c1, u32 p0, u32 p1, u64* tern, bool accumulate) {
  constexpr int TPP = TE / EPT;
  const u32 m = c->full;
  const u32 pairs = p1 - p0;
  const u32 groups = (pairs + 255) / 256;
  const u32 per_cta = (pairs + groups - 1) / groups;
  const u32 threads = std::max<u32>(64, ((per_cta * TPP + 31) / 32) * 32);
  need(n * TE <= 4 * threads, LCL_SHAPE_ERROR, "too many clients for one tile");
  dim3 grid((u32)(m * c->n / TE), groups);
  const size_t smem = (size_t)STAGES * n * (2 * TE + 2) * 8;
  need(smem <= 200 * 1024, LCL_SHAPE_ERROR, "too many clients for one tile");
  allow_smem(pair_accumulate<TE, EPT, STAGES>, smem);
  ProfScope ps(c, "pair_accumulate",
               8.0 * c->N() * m * (2.0 * n * (c1 - c0) * groups + 3.0 * pairs * (accumulate ? 2 : 1)));
  pair_accumulate<TE, EPT, STAGES><<<grid, threads, smem, c->stream>>>(
      clients, n, c0, c1, chunks, m, c->logn, c->d_pairs, p0, p1, per_cta, tern,
      accumulate ? 1 : 0, c->d_primes);
  post_launch(c);
}

// Pairs one accumulation launch covers: the i<j row-major range [a, b) of
// the matrix (kind 0), or every pair (i, j), i < j, with j in [a, b) in
// j-major order (kind 1: the pairs completed once clients [0, b) have
// arrived, see lcl_server_round_host). Output index = position in the set.
struct PairSet {
  u32 a, b, kind;
};
PairSet row_range(u32 p0, u32 p1) { return PairSet{p0, p1, 0}; }
PairSet completed_by(u32 j0, u32 j1) { return PairSet{j0, j1, 1}; }

std::vector<uint2> pair_list(u32 n, const PairSet& ps) {
  std::vector<uint2> all;
  if (ps.kind == 1) {
    for (u32 j = ps.a; j < ps.b && j < n; ++j)
      for (u32 i = 0; i < j; ++i) all.push_back(make_uint2(i | (j << 16), (u32)all.size()));
    return all;
  }
  u32 p = 0;
  for (u32 i = 0; i < n; ++i)
    for (u32 j = i + 1; j < n; ++j, ++p)
      if (p >= ps.a && p < ps.b) all.push_back(make_uint2(i | (j << 16), p - ps.a));
  return all;
}
u32 pair_count(u32 n, const PairSet& ps) {
  if (ps.kind == 0) return ps.b - ps.a;
  const u64 hi = std::min(ps.b, n), lo = std::min(ps.a, n);
  return (u32)(hi * (hi - 1) / 2 - lo * (lo - 1) / 2);  // lo = 0: 0 * (2^64 - 1) = 0
}

// Bank-aware pair schedule for pair_accumulate_f64 (TPP = 1): the set cut
// into CTA groups of per_cta; inside a group, every quarter warp (8 threads,
// one 16-byte shared-memory wavefront) gets pairs whose i's and j's fall in
// distinct bank groups (client k's tile row starts at 16-byte unit
// k * CS / 2, CS / 2 odd), greedily.
// Orders one CTA's pairs so that every 8 consecutive threads (a quarter warp
// of 16-byte shared-memory reads) touch clients of distinct bank groups
// ((client * cs_half) mod 8) where possible; appends to out.
void bank_order(std::vector<uint2> rem, u32 cs_half, std::vector<uint2>& out) {
  while (!rem.empty()) {
    int ib[8], jb[8];
    for (int b = 0; b < 8; ++b) ib[b] = jb[b] = -1;
    std::vector<uint2> grp, rest;
    for (const uint2& e : rem) {
      const int i = e.x & 0xFFFF, j = e.x >> 16;
      const int bi = (int)((i * cs_half) % 8), bj = (int)((j * cs_half) % 8);
      if (grp.size() < 8 && (ib[bi] < 0 || ib[bi] == i) && (jb[bj] < 0 || jb[bj] == j)) {
        ib[bi] = i;
        jb[bj] = j;
        grp.push_back(e);
      } else {
        rest.push_back(e);
      }
    }
    while (grp.size() < 8 && !rest.empty()) {  // no conflict-free pair left: accept one
      grp.push_back(rest.front());
      rest.erase(rest.begin());
    }
    out.insert(out.end(), grp.begin(), grp.end());
    rem.swap(rest);
  }
}

// Client-blocked pair groups for the full pair set of n clients: clients in
// blocks of kPairBlock; one group per off-diagonal block pair (I < J: all
// pairs across, 2 blocks staged) and one per two diagonal blocks (the pairs
// inside each), so a CTA stages <= 2 * kPairBlock clients per chunk instead
// of all n. Device layout: [groups * per_cta] uint2 entries (local client
// indices, output pair index; .y = ~0 pads), then [groups * nl] u16 client
// lists (padded with the group's first client).
constexpr u32 kPairBlock = 13;  // 13 x 13 = 169 pairs <= 192 threads
struct BlockedSchedule {
  const uint2* sched;
  const unsigned short* clist;
  u32 groups, per_cta, nl;
};
BlockedSchedule pair_schedule_blocked(lcl_context* c, u32 n, u32 cs_half, const PairSet& ps) {
  std::vector<std::vector<u32>> blocks;
  for (u32 b0 = 0; b0 < n; b0 += kPairBlock) {
    blocks.emplace_back();
    for (u32 i = b0; i < std::min(n, b0 + kPairBlock); ++i) blocks.back().push_back(i);
  }
  std::vector<std::vector<u32>> cls;  // clients of each group
  const u32 nb = (u32)blocks.size();
  for (u32 I = 0; I < nb; ++I)
    for (u32 J = I + 1; J < nb; ++J) {
      cls.push_back(blocks[I]);
      cls.back().insert(cls.back().end(), blocks[J].begin(), blocks[J].end());
    }
  std::vector<u32> diag_groups;  // index into cls of groups made of diagonal blocks
  for (u32 I = 0; I < nb; I += 2) {
    diag_groups.push_back((u32)cls.size());
    cls.push_back(blocks[I]);
    if (I + 1 < nb) cls.back().insert(cls.back().end(), blocks[I + 1].begin(), blocks[I + 1].end());
  }
  // pairs of each group, output index = row-major pair number
  std::vector<std::vector<uint2>> prs(cls.size());
  std::vector<u32> blk(n);
  for (u32 I = 0; I < nb; ++I)
    for (u32 i : blocks[I]) blk[i] = I;
  auto group_of = [&](u32 I, u32 J) {  // I <= J
    if (I == J) return diag_groups[I / 2];
    return I * nb - I * (I + 1) / 2 + (J - I - 1);
  };
  auto local = [&](u32 g, u32 i) {
    return (u32)(std::find(cls[g].begin(), cls[g].end(), i) - cls[g].begin());
  };
  // output index of pair (i, j) in the set, or -1 (row-major range [a, b),
  // or the j-major pairs of clients j in [a, b))
  auto out_index = [&](u64 i, u64 j, u64 p) -> long long {
    if (ps.kind == 0) return p >= ps.a && p < ps.b ? (long long)(p - ps.a) : -1;
    if (j < ps.a || j >= ps.b) return -1;
    return (long long)(j * (j - 1) / 2 - (u64)ps.a * (ps.a ? ps.a - 1 : 0) / 2 + i);
  };
  u64 p = 0;
  for (u32 i = 0; i < n; ++i)
    for (u32 j = i + 1; j < n; ++j, ++p) {
      const long long o = out_index(i, j, p);
      if (o < 0) continue;
      const u32 g = group_of(blk[i], blk[j]);
      prs[g].push_back(make_uint2(local(g, i) | (local(g, j) << 16), (u32)o));
    }
  {  // only groups with pairs of the set launch
    std::vector<std::vector<u32>> c2;
    std::vector<std::vector<uint2>> p2;
    for (size_t g = 0; g < cls.size(); ++g)
      if (!prs[g].empty()) {
        c2.push_back(cls[g]);
        p2.push_back(prs[g]);
      }
    cls.swap(c2);
    prs.swap(p2);
  }
  u32 per_cta = 0, nl = 0;
  for (size_t g = 0; g < cls.size(); ++g) {
    per_cta = std::max<u32>(per_cta, (u32)prs[g].size());
    nl = std::max<u32>(nl, (u32)cls[g].size());
  }
  const u32 groups = (u32)cls.size();
  const auto key = std::make_tuple(n | (1u << 30) | (ps.kind << 31), ps.a, ps.b, cs_half);
  auto it = c->sched.find(key);
  if (it != c->sched.end()) {
    return {it->second, reinterpret_cast<const unsigned short*>(it->second + (size_t)groups * per_cta), groups,
            per_cta, nl};
  }
  std::vector<uint2> out;
  for (u32 g = 0; g < groups; ++g) {
    const size_t before = out.size();
    bank_order(prs[g], cs_half, out);
    out.resize(before + per_cta, make_uint2(0u, ~0u));
  }
  std::vector<unsigned short> cl((size_t)groups * nl);
  for (u32 g = 0; g < groups; ++g)
    for (u32 t = 0; t < nl; ++t) cl[(size_t)g * nl + t] = (unsigned short)(t < cls[g].size() ? cls[g][t] : cls[g][0]);
  const size_t sbytes = out.size() * sizeof(uint2);
  uint2* d = nullptr;
  cuda_check(cudaMalloc(&d, sbytes + cl.size() * sizeof(unsigned short)), "schedule alloc");
  cuda_check(cudaMemcpy(d, out.data(), sbytes, cudaMemcpyHostToDevice), "schedule upload");
  cuda_check(cudaMemcpy(reinterpret_cast<char*>(d) + sbytes, cl.data(), cl.size() * sizeof(unsigned short),
                        cudaMemcpyHostToDevice),
             "schedule upload");
  c->sched[key] = d;
  return {d, reinterpret_cast<const unsigned short*>(d + (size_t)groups * per_cta), groups, per_cta, nl};
}

const uint2* pair_schedule(lcl_context* c, u32 n, const PairSet& ps, u32 per_cta, u32 cs_half) {
  const auto key = std::make_tuple(n | (ps.kind << 31), ps.a, ps.b, per_cta * 64 + cs_half);
  auto it = c->sched.find(key);
  if (it != c->sched.end()) return it->second;
  const std::vector<uint2> all = pair_list(n, ps);
  std::vector<uint2> out;
  out.reserve(all.size());
  for (size_t g0 = 0; g0 < all.size(); g0 += per_cta) {
    bank_order(std::vector<uint2>(all.begin() + g0, all.begin() + std::min(all.size(), (size_t)g0 + per_cta)),
               cs_half, out);
  }
  uint2* d = nullptr;
  cuda_check(cudaMalloc(&d, out.size() * sizeof(uint2)), "schedule alloc");
  cuda_check(cudaMemcpy(d, out.data(), out.size() * sizeof(uint2), cudaMemcpyHostToDevice),
             "schedule upload");
  c->sched[key] = d;
  return d;
}

template <int TE, int STAGES, int MINB, bool PF, int W = 1>
bool pair_accumulate_f64_cfg(lcl_context* c, const u64* clients, u32 n, u32 chunks, u32 c0,
                             u32 c1, const PairSet& ps, u64* tern, bool accumulate) {
  constexpr int MAXT = 192;
  static_assert(kPairBlock * kPairBlock <= MAXT, "an off-diagonal block pair fills one CTA");
  const u32 m = c->full;
  const u32 pairs = pair_count(n, ps);
  // client-blocked groups once n exceeds two blocks, for any pair set (whole
  // matrix, a sub-batch or shard range, or a host-round group), so a CTA
  // never stages more than 2 * kPairBlock clients (LCL_PAIR_BLOCKED=0 turns
  // them off)
  const char* eb = std::getenv("LCL_PAIR_BLOCKED");
  const bool blocked = n > 2 * kPairBlock + 1 && !(eb && eb[0] == '0');
  u32 groups = (pairs + MAXT - 1) / MAXT;
  u32 per_cta = (pairs + groups - 1) / groups;
  u32 nl = n, sched_len = pairs;
  const uint2* sched = nullptr;
  const unsigned short* clist = nullptr;
  if (blocked) {
    const BlockedSchedule bs = pair_schedule_blocked(c, n, TE + 1, ps);
    sched = bs.sched;
    clist = bs.clist;
    groups = bs.groups;
    per_cta = bs.per_cta;
    nl = bs.nl;
    sched_len = groups * per_cta;
  }
  // every warp of a CTA runs the pair math (warps of padding included), so
  // the CTA is sized to the schedule: one warp for <= 32 pairs (a host-round
  // group of one client) -- LCL_PAIR_MIN_THREADS (default 32; 64 before)
  static const u32 min_threads = [] {
    const char* e = std::getenv("LCL_PAIR_MIN_THREADS");
    return e ? (u32)std::max(32, atoi(e)) : 32u;
  }();
  u32 threads = std::max<u32>(min_threads, ((per_cta + 31) / 32) * 32);
  if (W > 1) {  // W warps on a W * TE-slot tile, one warp's worth of pairs
    if (blocked || per_cta > 32) return false;
    threads = 32 * W;
  }
  const size_t smem = (size_t)STAGES * W * nl * (2 * TE + 2) * 8;
  if (smem > 100 * 1024) return false;
  if (!blocked) sched = pair_schedule(c, n, ps, per_cta, TE + 1);
  const u64 tiles = (u64)m * c->n / (TE * W);
  allow_smem(pair_accumulate_f64<TE, STAGES, MAXT, MINB, PF, W>, smem);
  for (u32 cb = c0; cb < c1; cb += 256) {  // exact for 256 chunks per pass
    const u32 ce = std::min(c1, cb + 256);
    const bool acc = accumulate || cb > c0;
    ProfScope ps(c, "pair_accumulate",
                 8.0 * c->N() * m * (2.0 * n * (ce - cb) * groups + 3.0 * pairs * (acc ? 2 : 1)));
    pair_accumulate_f64<TE, STAGES, MAXT, MINB, PF, W><<<(u32)(tiles * groups), threads, smem, c->stream>>>(
        clients, n, cb, ce, chunks, m, c->logn, sched, sched_len, groups, per_cta, tern, acc ? 1 : 0,
        c->d_primes, clist, nl);
    post_launch(c);
  }
  return true;
}

// pair_accumulate on the FP64 pipe when the q-chain allows it (measured at
// cfg3, 190 pairs x 342 chunks: <8,6,2,false> 26.2 ms, <4,8,3,false> 27.9,
// <4,8,2,true> 30.0, <2,8,4,false> 45.7; split-23 integer kernel 50.3; a
// warp-specialised variant -- producer warp, full/empty mbarriers, no CTA
// barrier -- ran 29.6 ms with cp.async and 55 ms with 64-byte TMA bulk
// copies, which are issue-bound at this row size; round 2: a client-quad
// form (a thread owns a 2 x 2 block of pairs {i1,i2} x {j1,j2}, half the
// staged words per pair-slot for the same FP64 work) ran 35.6 ms with one
// slot per thread (400 threads, 1 CTA/SM) and 36.3 ms with two (128
// registers, 2 CTAs/SM) against 25.4 ms -- parity-green, not kept; a
// dual-pipe form putting 25 / 40 / 55 % of each CTA's pairs on the integer
// multiply pipe (split-23 sums, two threads per pair, warp-uniform roles)
// ran 34.3 / 37.1 / 37.5 ms -- the two roles' staging share one L1 and the
// integer products cost ~2x the FP64 ones; OR-ing the exponent into the
// staged tile once per CTA (by each vector's copying thread, before the
// barrier) instead of once per pair ran 26.7-27.0 vs 25.5-25.7 ms),
// else the split-23 integer kernel.
void pair_accumulate_launch(lcl_context* c, const u64* clients, u32 n, u32 chunks, u32 c0,
                            u32 c1, const PairSet& ps, u64* tern, bool accumulate) {
  // <= 32 pairs (a host-round group of one client): 4 warps on a 32-slot
  // tile, 256-byte copies (LCL_PAIR_W=1 turns it off)
  const char* we = std::getenv("LCL_PAIR_W");
  const int pw = we ? atoi(we) : 4;
  if (c->pair_f64 && pw == 4 && c->n >= 32 * 8 &&
      pair_accumulate_f64_cfg<8, 6, 2, false, 4>(c, clients, n, chunks, c0, c1, ps, tern, accumulate))
    return;
  if (c->pair_f64 && pw == 2 && c->n >= 16 * 8 &&
      pair_accumulate_f64_cfg<8, 6, 2, false, 2>(c, clients, n, chunks, c0, c1, ps, tern, accumulate))
    return;
  if (c->pair_f64 &&
      pair_accumulate_f64_cfg<8, 6, 2, false>(c, clients, n, chunks, c0, c1, ps, tern, accumulate))
    return;
  need(ps.kind == 0, LCL_USAGE_ERROR, "j-major pair sets need the FP64 accumulation kernel");
  pair_accumulate_cfg<8, 4, 8>(c, clients, n, chunks, c0, c1, ps.a, ps.b, tern, accumulate);
}

// ------------------------------------------------------------ KGC decode
// Embedding tables of the reference (encoding.cpp:40-80): twist[i] =
// polar(1, pi i / N), roots[k] = polar(1, 2 pi k / h), the bit reversal of
// log2 h bits and slot_index[j] = (5^j mod 2N - 1) / 4, computed with the same
// host libm expressions, so the device FFT sees the reference's doubles.
void ensure_decode_tables(lcl_context* c) {
  if (c->d_twist) return;
  const size_t n = c->n, h = n / 2;
  const int logh = __builtin_ctzll(h);
  const double pi = 3.141592653589793238462643383279502884;  // std::numbers::pi
  std::vector<double2> tw(h), rt(h / 2 > 0 ? h / 2 : 1);
  for (size_t i = 0; i < h; ++i) {
    const double ang = pi * static_cast<double>(i) / static_cast<double>(n);
    tw[i] = make_double2(std::cos(ang), std::sin(ang));
  }
  for (size_t k = 0; k < h / 2; ++k) {
    const double ang = 2.0 * pi * static_cast<double>(k) / static_cast<double>(h);
    rt[k] = make_double2(std::cos(ang), std::sin(ang));
  }
  std::vector<u32> brv(h), slot(h);
  for (size_t i = 0; i < h; ++i) brv[i] = (u32)h_brv(i, logh);
  u64 g = 1;
  for (size_t j = 0; j < h; ++j) {
    slot[j] = (u32)((g - 1) / 4);
    g = (g * 5) % (2 * n);
  }
  cuda_check(cudaMalloc(&c->d_twist, h * sizeof(double2)), "alloc");
  cuda_check(cudaMalloc(&c->d_roots, rt.size() * sizeof(double2)), "alloc");
  cuda_check(cudaMalloc(&c->d_brv, h * 4), "alloc");
  cuda_check(cudaMalloc(&c->d_slot, h * 4), "alloc");
  cuda_check(cudaMemcpy(c->d_twist, tw.data(), h * sizeof(double2), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_roots, rt.data(), rt.size() * sizeof(double2), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_brv, brv.data(), h * 4, cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_slot, slot.data(), h * 4, cudaMemcpyHostToDevice), "upload");
}

// decrypt (ckks.cpp:381-388): pt [B][m][N] = c1 * s + c0, evaluation domain.
void decrypt_batch(lcl_context* c, const u64* ct, u32 B, u32 m, const u64* sk, u64* pt) {
  const u64 total = (u64)B * m * c->N();
  if (!total) return;
  ProfScope ps(c, "decrypt_rows", 8.0 * (double)total * 4);
  decrypt_rows<<<(u32)((total + 255) / 256), 256, 0, c->stream>>>(ct, sk, B, m, c->logn, pt,
                                                                  c->d_primes);
  post_launch(c);
}

// decode (ckks.cpp:313-348 + encoding.cpp:118-134) of B plaintexts [B][m][N]
// in the evaluation domain (transformed in place to coefficients) into
// slots [B][N/2] doubles.
void decode_batch(lcl_context* c, u64* pt, u32 B, u32 m, double scale, double* slots) {
  if (B == 0) return;
  need(m >= 1 && m <= c->full, LCL_SHAPE_ERROR, "plaintext level outside the chain");
  ensure_decode_tables(c);
  const u64 N = c->N();
  const u32 h = (u32)(N / 2), logh = (u32)c->logn - 1;
  const RowMap rows = make_map(pt, m, N, (u64)m * N, 1, 0, c->primes_0(m));
  launch_inv(c, B * m, rows, PlainStore{rows});
  CrtConst k;
  k.q0 = c->primes[0];
  k.q1 = m >= 2 ? c->primes[1] : 1;
  k.inv01 = m >= 2 ? h_invmod(k.q0 % k.q1, k.q1) : 0;
  k.inv01s = m >= 2 ? h_shoup(k.inv01, k.q1) : 0;
  double2* bk = reinterpret_cast<double2*>(c->ws_dec.get((u64)B * h * 2));
  const u64 tot = (u64)B * h;
  {
    ProfScope ps(c, "decode_twist", 8.0 * (double)tot * (2.0 * std::min<u32>(m, 2) + 2));
    decode_twist<<<(u32)((tot + 255) / 256), 256, 0, c->stream>>>(pt, B, m, (u32)c->logn, k, scale,
                                                                  c->d_twist, c->d_brv, bk);
    post_launch(c);
  }
  {
    const u32 bs = std::min<u32>(h, 256);
    ProfScope ps(c, "fft_blocks", 32.0 * (double)tot);
    fft_blocks<<<(u32)(tot / bs), 128, 0, c->stream>>>(bk, logh, c->d_roots);
    post_launch(c);
  }
  if (h > 256) {
    const size_t smem = (size_t)(h / 256) * 16 * sizeof(double2);
    allow_smem(fft_columns, smem);
    ProfScope ps(c, "fft_columns", 32.0 * (double)tot);
    fft_columns<<<B * 16, 256, smem, c->stream>>>(bk, logh, c->d_roots);
    post_launch(c);
  }
  {
    ProfScope ps(c, "decode_slots", 24.0 * (double)tot);
    decode_slots<<<(u32)((tot + 255) / 256), 256, 0, c->stream>>>(bk, B, logh, c->d_slot, slots);
    post_launch(c);
  }
}

// ------------------------------------------------------------ client encryption
// pack_and_encrypt (distance.cpp:64-91) of one client's weights: per chunk,
// in the reference's draw order, r (sample_secret_like: sparse ternary of
// Hamming weight 64, ckks.cpp:187-193), e0 and e1 (CBD, eta 21) from the
// client's Sampler; the encodings (slots_to_coeffs + rounding, a pure
// function of the weights) run on host threads meanwhile; then one batched
// device pass lifts, transforms and combines with the public key.
constexpr size_t kHammingWeight = 64;  // CkksParams::key_hamming_weight (ckks.hpp:48)
constexpr int kErrorEta = 21;          // CkksParams::error_eta (ckks.hpp:50)
constexpr double kMessageBound = 1048576.0;  // CkksParams::message_bound = 2^20

// encode + encrypt (ckks.cpp:263-307, 350-379) of V value vectors, in order,
// into out [V][2][full][N]: vec(v) -> (pointer, length) of vector v.
template <class Vec>
void encrypt_vectors(lcl_context* c, lcl_sampler* rng, size_t V, const Vec& vec, const u64* pk,
                     u64* out) {
  const size_t n = c->n;
  const u32 m = c->full;
  for (size_t v = 0; v < V; ++v) {  // the reference's encode checks (ckks.cpp:267-281)
    const auto [p, len] = vec(v);
    need(len <= n / 2, LCL_CAPACITY_ERROR, "more values than slots");
    for (size_t i = 0; i < len; ++i)
      need(std::isfinite(p[i]) && std::fabs(p[i]) <= kMessageBound, LCL_CAPACITY_ERROR,
           "value outside the message bound");
  }
  std::vector<long long> rounded(V * n);
  std::vector<signed char> small(V * 3 * n);
  {
    // encodings on worker threads (independent of the draws)
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 16));
    std::vector<std::thread> pool;
    std::vector<std::string> err(nt);
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        try {
          for (size_t v = t; v < V; v += nt) {
            const auto [p, len] = vec(v);
            const std::vector<long long> r = h_encode_rounded(std::vector<double>(p, p + len), n, c->scale);
            std::copy(r.begin(), r.end(), rounded.begin() + v * n);
          }
        } catch (const LclError& e) {
          err[t] = e.msg;
        }
      });
    // the draws, sequentially, in the reference's order
    for (size_t v = 0; v < V; ++v) {
      signed char* s = small.data() + v * 3 * n;
      if (kHammingWeight == 0)
        rng->ternary(n, s);
      else
        rng->sparse_ternary(n, kHammingWeight, s);
      rng->cbd(n, kErrorEta, s + n);
      rng->cbd(n, kErrorEta, s + 2 * n);
    }
    for (auto& th : pool) th.join();
    for (auto& e : err) need(e.empty(), LCL_CAPACITY_ERROR, e.empty() ? "" : e.c_str());
  }
  const u64 N = c->N();
  const size_t batch = std::max<size_t>(1, std::min<size_t>(V, (size_t)((2ull << 30) / (4 * m * N * 8))));
  for (size_t c0 = 0; c0 < V; c0 += batch) {
    const u32 B = (u32)std::min(batch, V - c0);
    u64* ws = c->ws_enc.get((u64)B * 4 * m * N);
    long long* d_round = reinterpret_cast<long long*>(c->ws_enc_in.get((u64)B * N + (B * 3 * N + 7) / 8));
    signed char* d_small = reinterpret_cast<signed char*>(d_round + (u64)B * N);
    cuda_check(cudaMemcpyAsync(d_round, rounded.data() + c0 * n, (u64)B * N * 8,
                               cudaMemcpyHostToDevice, c->stream), "h2d");
    cuda_check(cudaMemcpyAsync(d_small, small.data() + c0 * 3 * n, (u64)B * 3 * N,
                               cudaMemcpyHostToDevice, c->stream), "h2d");
    const u64 total = (u64)B * m * N;
    {
      ProfScope ps(c, "encrypt_lift", (double)B * N * 11 + 8.0 * total * 4);
      encrypt_lift<<<(u32)((total + 255) / 256), 256, 0, c->stream>>>(d_round, d_small, B, m,
                                                                      c->logn, ws, c->d_primes);
      post_launch(c);
    }
    const RowMap wm = make_map(ws, m, N, (u64)m * N, 1, 0, c->primes_0(m));
    launch_fwd(c, B * 4 * m, wm, PlainLoad{wm}, PlainStore{wm});
    {
      ProfScope ps(c, "encrypt_combine", 8.0 * total * 8);
      encrypt_combine<<<(u32)((total + 255) / 256), 256, 0, c->stream>>>(
          ws, pk, B, m, c->logn, out + c0 * 2 * m * N, c->d_primes);
      post_launch(c);
    }
    // the host staging must outlive the copies
    cuda_check(cudaStreamSynchronize(c->stream), "encrypt");
  }
  c->counts.encryptions += V;
}

void pack_and_encrypt(lcl_context* c, lcl_sampler* rng, const double* w, size_t dim,
                      double prescale, const u64* pk, u64* out) {
  need(dim > 0, LCL_SHAPE_ERROR, "empty weight vector");
  need(prescale > 0.0 && std::isfinite(prescale), LCL_PARAMETER_ERROR,
       "prescale must be positive and finite");
  for (size_t i = 0; i < dim; ++i) need(std::isfinite(w[i]), LCL_DATA_ERROR, "weights must be finite");
  const size_t slots = c->n / 2;
  const size_t C = (dim + slots - 1) / slots;
  std::vector<double> scaled(w, w + dim);
  for (double& v : scaled) v *= prescale;
  encrypt_vectors(c, rng, C, [&](size_t ch) {
    const size_t lo = ch * slots;
    return std::pair<const double*, size_t>(scaled.data() + lo, std::min(slots, dim - lo));
  }, pk, out);
}

// generate_keys (ckks.cpp:225-261): the draws on the host in the reference's
// order (secret, public a and e, then for every switch key and digit a and
// e), the transforms and products on the device. Rotation keys for the
// distinct nonzero steps mod slots, in the caller's order.
struct KeygenScratch {
  u64* a;
  u64* e;
  signed char* small;
};

void keygen_uniform(lcl_context* c, lcl_sampler* rng, u32 rows, std::vector<u64>& h) {
  const size_t n = c->n;
  h.resize((size_t)rows * n);
  for (u32 r = 0; r < rows; ++r) {  // uniform_poly, row by row (sampling.cpp:47-55)
    const u64 q = c->primes[r < c->full ? r : c->full];
    for (size_t i = 0; i < n; ++i) h[(size_t)r * n + i] = rng->uniform_below(q);
  }
}

// e (CBD) over `rows` rows into the evaluation domain at d_e
void keygen_error(lcl_context* c, lcl_sampler* rng, u32 rows, const KeygenScratch& ks,
                  std::vector<signed char>& hs) {
  const size_t n = c->n;
  hs.resize(n);
  rng->cbd(n, kErrorEta, hs.data());
  cuda_check(cudaMemcpyAsync(ks.small, hs.data(), n, cudaMemcpyHostToDevice, c->stream), "h2d");
  const u64 tot = (u64)rows * n;
  lift_small<<<(u32)((tot + 255) / 256), 256, 0, c->stream>>>(ks.small, rows, c->logn, c->full,
                                                              ks.e, c->d_primes);
  post_launch(c);
  std::vector<u32> pr(rows);
  for (u32 r = 0; r < rows; ++r) pr[r] = r < c->full ? r : c->full;
  const RowMap em = make_map(ks.e, rows, c->N(), (u64)rows * c->N(), 1, 0, pr);
  launch_fwd(c, rows, em, PlainLoad{em}, PlainStore{em});
}

// make_switch_key (ckks.cpp:195-223) of target [(full+1)][N] into key
// [full][2][full+1][N].
void keygen_switch_key(lcl_context* c, lcl_sampler* rng, const u64* d_target, const u64* d_sk,
                       const KeygenScratch& ks, u64* key) {
  const u32 full = c->full, rows = full + 1;
  const u64 N = c->N(), tot = (u64)rows * N;
  std::vector<u64> ha;
  std::vector<signed char> hs;
  for (u32 j = 0; j < full; ++j) {
    u64* k0 = key + (u64)j * 2 * tot;
    u64* a = k0 + tot;
    keygen_uniform(c, rng, rows, ha);
    cuda_check(cudaMemcpyAsync(a, ha.data(), tot * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
    keygen_error(c, rng, rows, ks, hs);
    const u64 theta = c->primes[full] % c->primes[j];
    key_rows<<<(u32)((tot + 255) / 256), 256, 0, c->stream>>>(a, d_sk, ks.e, rows, c->logn,
                                                             d_target, j, theta, k0, c->d_primes);
    post_launch(c);
    // ha / hs are reused by the next digit: the copies must have landed
    cuda_check(cudaStreamSynchronize(c->stream), "keygen");
  }
}

std::vector<u32> galois_perm(size_t n, int logn, size_t step);  // rns.cpp:508-532, below

size_t generate_keys(lcl_context* c, lcl_sampler* rng, const size_t* steps, size_t nsteps,
                     u64* d_sk, u64* d_pk, u64* d_relin, u64* d_rot, size_t* rot_steps) {
  const u32 full = c->full, rows = full + 1;
  const size_t n = c->n;
  const u64 N = c->N();
  KeygenScratch ks;
  ks.a = nullptr;
  ks.e = c->ws_enc.get((u64)rows * N);
  ks.small = reinterpret_cast<signed char*>(c->ws_enc_in.get((n + 7) / 8));
  std::vector<signed char> hs(n);
  std::vector<u64> ha;
  // secret: sample_secret_like over full + 1 rows, then forward NTT
  if (kHammingWeight == 0)
    rng->ternary(n, hs.data());
  else
    rng->sparse_ternary(n, kHammingWeight, hs.data());
  cuda_check(cudaMemcpyAsync(ks.small, hs.data(), n, cudaMemcpyHostToDevice, c->stream), "h2d");
  lift_small<<<(u32)(((u64)rows * N + 255) / 256), 256, 0, c->stream>>>(ks.small, rows, c->logn,
                                                                        full, d_sk, c->d_primes);
  post_launch(c);
  std::vector<u32> pr(rows);
  for (u32 r = 0; r < rows; ++r) pr[r] = r < full ? r : full;
  const RowMap skm = make_map(d_sk, rows, N, (u64)rows * N, 1, 0, pr);
  launch_fwd(c, rows, skm, PlainLoad{skm}, PlainStore{skm});
  cuda_check(cudaStreamSynchronize(c->stream), "keygen");
  // public key: a uniform over the full q rows, e, p0 = -a s + e, p1 = a
  keygen_uniform(c, rng, full, ha);
  u64* p1 = d_pk + (u64)full * N;
  cuda_check(cudaMemcpyAsync(p1, ha.data(), (u64)full * N * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
  keygen_error(c, rng, full, ks, hs);
  key_rows<<<(u32)(((u64)full * N + 255) / 256), 256, 0, c->stream>>>(
      p1, d_sk, ks.e, full, c->logn, nullptr, 0, 0, d_pk, c->d_primes);
  post_launch(c);
  cuda_check(cudaStreamSynchronize(c->stream), "keygen");
  // relinearization key: target s^2
  u64* tgt = c->ws_pt.get((u64)rows * N);
  square_rows<<<(u32)(((u64)rows * N + 255) / 256), 256, 0, c->stream>>>(d_sk, rows, c->logn, tgt,
                                                                         c->d_primes);
  post_launch(c);
  keygen_switch_key(c, rng, tgt, d_sk, ks, d_relin);
  // rotation keys: target apply_galois(s, elt(step))
  const u64 kw = (u64)full * 2 * rows * N;
  size_t nk = 0;
  std::vector<size_t> done;
  u32* dperm = reinterpret_cast<u32*>(c->ws_dec.get((n + 1) / 2));
  for (size_t i = 0; i < nsteps; ++i) {
    const size_t st = steps[i] % (n / 2);
    if (st == 0 || std::find(done.begin(), done.end(), st) != done.end()) continue;
    done.push_back(st);
    const std::vector<u32> perm = galois_perm(n, c->logn, st);
    cuda_check(cudaMemcpyAsync(dperm, perm.data(), n * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
    permute_rows<<<(u32)(((u64)rows * N + 255) / 256), 256, 0, c->stream>>>(d_sk, dperm, rows,
                                                                            c->logn, tgt);
    post_launch(c);
    keygen_switch_key(c, rng, tgt, d_sk, ks, d_rot + nk * kw);
    if (rot_steps) rot_steps[nk] = st;
    ++nk;
  }
  return nk;
}

// build_mask (aggregation.cpp:156-186): n rank rows (basis vectors of the
// selected indices, in rank order) then n broadcast client selectors.
void build_mask(lcl_context* c, lcl_sampler* rng, size_t n, const size_t* selected, size_t l,
                const u64* pk, u64* rank_rows, u64* selectors) {
  need(n <= c->n / 2, LCL_CAPACITY_ERROR, "more clients than mask slots");
  for (size_t i = 0; i < l; ++i)
    need(selected[i] < n, LCL_SHAPE_ERROR, "selected index outside the client range");
  std::vector<double> rows(n * n, 0.0), sel(n * (c->n / 2), 0.0);
  for (size_t r = 0; r < n && r < l; ++r) rows[r * n + selected[r]] = 1.0;
  std::vector<bool> chosen(n, false);
  for (size_t i = 0; i < l; ++i) chosen[selected[i]] = true;
  for (size_t i = 0; i < n; ++i)
    std::fill(sel.begin() + i * (c->n / 2), sel.begin() + (i + 1) * (c->n / 2), chosen[i] ? 1.0 : 0.0);
  encrypt_vectors(c, rng, n, [&](size_t r) {
    return std::pair<const double*, size_t>(rows.data() + r * n, n);
  }, pk, rank_rows);
  encrypt_vectors(c, rng, n, [&](size_t i) {
    return std::pair<const double*, size_t>(sel.data() + i * (c->n / 2), c->n / 2);
  }, pk, selectors);
}

void hadd_into(lcl_context* c, u64* acc, const u64* x, u32 B, u32 m) {
  const u64 N = c->N();
  const RowMap a = ct_map(acc, m, N, 2ull * m * N);
  const RowMap b = ct_map(x, m, N, 2ull * m * N);
  const u32 rows = B * 2 * m;
  ProfScope ps(c, "hadd", 24.0 * N * rows);
  rows_addsub<false><<<(u32)(((u64)rows * N + 255) / 256), 256, 0, c->stream>>>(
      a, a, b, rows, c->logn, c->d_primes);
  post_launch(c);
  c->counts.additions += B;
}

// Sub-batch size for the key-switch chain: bounds the digit workspace.
u32 sub_batch(lcl_context* c, u32 m) {
  const u64 per_item = (u64)m * (m + 1) * c->N() * 8 * 2;  // digits + mid
  const u64 budget = 8ull << 30;
  return (u32)std::max<u64>(1, std::min<u64>(1024, budget / per_item));
}

// build_distance_matrix per_pair (distance.cpp:242-300), pairs in i<j order.
// Pairs [pair_begin, pair_end) of the (i<j) row-major order; out holds just
// that range (a shard of the matrix when the pairs are split across GPUs).
void distance_matrix(lcl_context* c, const u64* clients, u32 n, u32 chunks, size_t width,
                     size_t k, bool lazy, bool reduce, u64* out, u32 pair_begin = 0,
                     u32 pair_end = 0xFFFFFFFFu) {
  if (n < 2) fail(LCL_SHAPE_ERROR, "pairwise distances need at least two clients");
  if (n > 65535) fail(LCL_SHAPE_ERROR, "too many clients");
  const u32 m = c->full;
  if (m < 2) fail(LCL_DEPTH_EXHAUSTED, "no prime left to rescale by");
  const u64 N = c->N();
  ensure_pairs(c, n);
  const u32 P = std::min<u32>(n * (n - 1) / 2, pair_end);
  need(pair_begin <= P, LCL_SHAPE_ERROR, "pair range outside the matrix");
  if (reduce) {
    if (width == 0 || (width & (width - 1))) fail(LCL_WIDTH_ERROR, "reduction width must be a power of two");
    if (width > c->n / 2) fail(LCL_WIDTH_ERROR, "reduction width exceeds the slot count");
  }
  const u32 SB = sub_batch(c, m);
  const u64 out_stride = 2ull * (m - 1) * N;
  const u64 tern_words = 3ull * m * N;
  // When more pairs than one key-switch sub-batch remain, the ternaries of
  // ALL of them are accumulated in one pass over the clients (one launch,
  // every pair group of a tile adjacent in the grid, so each client tile
  // leaves HBM once), and only relinearisation / rescale / reduction run per
  // sub-batch: 3 sub-batches at 50 clients would otherwise re-stream the
  // clients 3 times with 137-pair CTAs instead of 175-pair ones.
  const u32 PA = P - pair_begin;
  const bool all_pairs = lazy && PA > SB && (u64)PA * tern_words * 8 <= (16ull << 30);
  u64* tern_all = nullptr;
  if (all_pairs) {
    tern_all = c->ws_tern.get((u64)PA * tern_words);
    for (u32 cb = 0; cb < chunks; cb += 32768)
      pair_accumulate_launch(c, clients, n, chunks, cb, std::min(chunks, cb + 32768),
                             row_range(pair_begin, P), tern_all, cb > 0);
  }
  for (u32 p0 = pair_begin; p0 < P; p0 += SB) {
    const u32 p1 = std::min(P, p0 + SB), B = p1 - p0;
    u64* o = out + (u64)(p0 - pair_begin) * out_stride;
    u64* ctA = c->ws_ctA.get((u64)B * 2 * m * N);
    if (lazy) {
      u64* tern = tern_all ? tern_all + (u64)(p0 - pair_begin) * tern_words
                           : c->ws_tern.get((u64)B * tern_words);
      if (!tern_all) {
        for (u32 cb = 0; cb < chunks; cb += 32768) {
          pair_accumulate_launch(c, clients, n, chunks, cb, std::min(chunks, cb + 32768),
                                 row_range(p0, p1), tern, cb > 0);
        }
      }
      relinearize_batch(c, tern, B, m, ctA);
      rescale_batch(c, ctA, B, m, o);
    } else {
      u64* tern = c->ws_tern.get((u64)B * 3 * m * N);
      u64* part = c->ws_ctB.get((u64)B * 2 * (m - 1) * N);
      for (u32 ch = 0; ch < chunks; ++ch) {
        pair_accumulate_launch(c, clients, n, chunks, ch, ch + 1, row_range(p0, p1), tern, false);
        relinearize_batch(c, tern, B, m, ctA);
        rescale_batch(c, ctA, B, m, ch == 0 ? o : part);
        if (ch) hadd_into(c, o, part, B, m - 1);
      }
    }
    // counters of the pair loop (hsub + hsquare + lazy_accumulate per chunk)
    c->counts.multiplications += (u64)B * chunks;
    c->counts.additions += (u64)B * (2ull * chunks - 1) - (lazy ? 0 : (u64)B * (chunks - 1));
    if (reduce) slot_reduce_batch(c, o, B, m - 1, width, k, o);
  }
}

void check_width(const lcl_context* c, size_t width) {
  if (width == 0 || (width & (width - 1))) fail(LCL_WIDTH_ERROR, "reduction width must be a power of two");
  if (width > c->n / 2) fail(LCL_WIDTH_ERROR, "reduction width exceeds the slot count");
}

// build_distance_matrix, DistanceMode::row_sums (distance.cpp:257-298): the
// pair distances are computed without a per-pair reduction (reduce_pairs is
// false in this mode), row i = the hadd chain of the n - 1 pairs containing
// client i (one launch for all rows), then one slot_reduce per row when
// reduce_on_server. out: [n][2][full-1][N].
void distance_rows(lcl_context* c, const u64* clients, u32 n, u32 chunks, size_t width, size_t k,
                   bool lazy, bool reduce, u64* out) {
  if (n < 2) fail(LCL_SHAPE_ERROR, "pairwise distances need at least two clients");
  if (reduce) {
    check_width(c, width);
    if (k == 0) fail(LCL_PARAMETER_ERROR, "unfold factor starts at 1");
  }
  const u32 m = c->full;
  if (m < 2) fail(LCL_DEPTH_EXHAUSTED, "no prime left to rescale by");
  const u64 N = c->N();
  const u64 P = (u64)n * (n - 1) / 2;
  const u64 W = 2ull * (m - 1) * N;
  u64* pairs = c->ws_rows.get(P * W);
  distance_matrix(c, clients, n, chunks, width, k, lazy, false, pairs);
  {
    ProfScope ps(c, "pair_row_sums", 8.0 * W * ((double)n * (n - 1) + n));
    const dim3 grid((u32)((W / 2 + 255) / 256), n);
    pair_row_sums<<<grid, 256, 0, c->stream>>>(pairs, n, m - 1, c->logn, out, c->d_primes);
    post_launch(c);
  }
  c->counts.additions += (u64)n * (n - 2);
  if (reduce) slot_reduce_batch(c, out, n, m - 1, width, k, out);
}

// Chunks [chunk_begin, chunk_end) of the aggregate (a shard when the chunks
// are split across GPUs); out holds just that range.
// encode(1/l at scale, level of the rescaled chunk) on the host
// (aggregation.cpp:221-223), NTT'd on the device and kept there per l, so
// repeated or sliced calls neither re-encode nor synchronise.
const u64* agg_plaintext(lcl_context* c, size_t l) {
  const u32 m = c->full;
  const u64 N = c->N();
  u64* d_pt = c->ws_ptl.get((u64)(m - 1) * N);
  if (c->pt_l != l) {
    std::vector<double> v(c->n / 2, 1.0 / (double)l);
    const std::vector<long long> rounded = h_encode_rounded(v, c->n, c->scale);
    c->pt_host.assign((u64)(m - 1) * N, 0);
    for (u32 r = 0; r < m - 1; ++r) {
      const u64 q = c->primes[r];
      for (u64 i = 0; i < N; ++i) {
        const long long x = rounded[i];
        const u64 mag = (u64)(x < 0 ? -x : x) % q;
        c->pt_host[r * N + i] = x < 0 ? (mag == 0 ? 0 : q - mag) : mag;
      }
    }
    // pt_host lives in the context, so the copy may stay asynchronous
    cuda_check(cudaMemcpyAsync(d_pt, c->pt_host.data(), c->pt_host.size() * 8,
                               cudaMemcpyHostToDevice, c->stream),
               "pt upload");
    const RowMap ptm = make_map(d_pt, m - 1, N, (u64)(m - 1) * N, 1, 0, c->primes_0(m - 1));
    launch_fwd(c, m - 1, ptm, PlainLoad{ptm}, PlainStore{ptm});
    c->pt_l = l;
  }
  return d_pt;
}

// Aggregate tensor of chunks [c0, c0 + B) over clients [i0, i1) into tern
// [B][3][m][N] (added mod q to its contents when accumulate).
void agg_tensor(lcl_context* c, const u64* clients, const u64* sel, u32 n, u32 chunks, u32 c0,
                u32 B, u32 i0, u32 i1, u64* tern, bool accumulate) {
  const u32 m = c->full;
  const u64 slots = (u64)m * c->N();
  constexpr int ST = 6;
  const size_t smem = (size_t)ST * 4 * 256 * 16;
  allow_smem(aggregate_stream<ST>, smem);
  // 2 slots per thread; min(256, N / 2) threads divide m * N / 2 for any m
  const u32 threads = (u32)std::min<u64>(256, c->N() / 2);
  ProfScope ps(c, "aggregate_tensor",
               8.0 * slots * (2.0 * (i1 - i0) * B + 2.0 * (i1 - i0) + 3.0 * B * (accumulate ? 2 : 1)));
  aggregate_stream<ST><<<(u32)(slots / 2 / threads * B), threads, smem, c->stream>>>(
      clients, sel, i0, i1, chunks, c0, B, m, c->logn, tern, accumulate ? 1 : 0, c->d_primes);
  post_launch(c);
  (void)n;
}

// relinearize + rescale (+ x encode(1/l) + rescale when averaging) of B
// aggregate ternaries into out [B][2][mo][N] (aggregation.cpp:218-224).
void agg_finish(lcl_context* c, const u64* tern, u32 B, bool average, const u64* d_pt, u64* out) {
  const u32 m = c->full;
  const u64 N = c->N();
  u64* ctA = c->ws_ctA.get((u64)B * 2 * m * N);
  relinearize_batch(c, tern, B, m, ctA);
  if (!average) {
    rescale_batch(c, ctA, B, m, out);
    return;
  }
  u64* ctB = c->ws_ctB.get((u64)B * 2 * (m - 1) * N);
  rescale_batch(c, ctA, B, m, ctB);
  const u64 total = (u64)B * 2 * (m - 1) * N;
  mult_plain<<<(u32)((total + 255) / 256), 256, 0, c->stream>>>(ctB, d_pt, B, m - 1, c->logn, ctB,
                                                                c->d_primes);
  post_launch(c);
  rescale_batch(c, ctB, B, m - 1, out);
  c->counts.multiplications += B;
}

void masked_aggregate(lcl_context* c, const u64* clients, const u64* sel, u32 n, u32 chunks,
                      size_t l, bool average, u64* out, u32 chunk_begin = 0,
                      u32 chunk_end = 0xFFFFFFFFu) {
  if (n == 0) fail(LCL_SHAPE_ERROR, "no client weights to aggregate");
  const u32 m = c->full;
  const u64 N = c->N();
  const u32 SB = sub_batch(c, m);
  const u32 mo = average ? m - 2 : m - 1;
  if (m < 2 || (average && m < 3)) fail(LCL_DEPTH_EXHAUSTED, "no prime left to rescale by");
  const u64* d_pt = average ? agg_plaintext(c, l) : nullptr;
  const u32 cend = std::min(chunks, chunk_end);
  need(chunk_begin <= cend, LCL_SHAPE_ERROR, "chunk range outside the weights");
  for (u32 c0 = chunk_begin; c0 < cend; c0 += SB) {
    const u32 c1 = std::min(cend, c0 + SB), B = c1 - c0;
    u64* tern = c->ws_tern.get((u64)B * 3 * m * N);
    agg_tensor(c, clients, sel, n, chunks, c0, B, 0, n, tern, false);
    agg_finish(c, tern, B, average, d_pt, out + (u64)(c0 - chunk_begin) * 2 * mo * N);
    c->counts.multiplications += (u64)n * B;
    c->counts.additions += (u64)(n - 1) * B;
  }
}

// CkksContext::hoisted_rotations (ckks.cpp:582-612) over B ciphertexts:
// one decomposition shared by every step; outs [nsteps][B][2][m][N].
void hoisted_batch(lcl_context* ctx, const u64* d_ct, u32 B, u32 m, const size_t* h_steps,
                   size_t nsteps, u64* d_outs) {
  const u64 N = ctx->N();
  const u64 words = (u64)B * 2 * m * N;
  std::vector<size_t> ks;     // nonzero steps, in order
  std::vector<size_t> where;  // their output slots
  for (size_t s = 0; s < nsteps; ++s) {
    const size_t st = norm_step(ctx, h_steps[s]);
    if (st == 0) {
      cuda_check(cudaMemcpyAsync(d_outs + s * words, d_ct, words * 8, cudaMemcpyDeviceToDevice,
                                 ctx->stream), "copy");
      continue;
    }
    if (!ctx->d_rot.count(st)) {
      // the reference throws here, after counting the decomposition and the
      // rotations of the steps before this one (ckks.cpp:595-611)
      if (!ks.empty()) {
        ctx->counts.mod_ups += B;
        ctx->counts.rotations += (u64)B * ks.size();
      }
      fail(LCL_KEY_ERROR, "no rotation key for the requested step");
    }
    ks.push_back(st);
    where.push_back(s);
  }
  if (ks.empty()) return;
  const RowMap c1 = make_map(d_ct + (u64)m * N, m, N, 2ull * m * N, 1, 0, ctx->primes_0(m));
  ctx->counts.mod_ups += B;
  ks_hoisted(ctx, c1, d_ct + (u64)m * N, 2ull * m * N, B, m, ks, [&](size_t i, u64* acc) {
    ks_moddown(ctx, acc, B, m, ct_map(d_outs + where[i] * words, m, N, 2ull * m * N), null_map(),
               ct_map(d_ct, m, N, 2ull * m * N), ctx->d_perm.at(ks[i]));
    ctx->counts.rotations += B;
  });
}

}  // namespace

// ============================================================ C-ABI
namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return LCL_OK;
  } catch (const LclError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return LCL_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return LCL_PARAMETER_ERROR;
  }
}


// Primes whose NTT rows run on the FP64 pipe (ntt.cuh FpF). Exactness needs
// q < 2^46 and every operand of f_mulmod below 2^51: forward inputs are below
// max(3q, q_s / 2) for the lift sources q_s of the same field, and 17 stages
// add at most 0.75q each. LCL_FP64=0 forces the integer field everywhere.
u32 fp_rows(const std::vector<u64>& primes) {
  const char* env = std::getenv("LCL_FP64");
  if (env && env[0] == '0') return 0;
  const u64 lim = 1ull << 46;
  u32 mask = 0;
  for (size_t d = 0; d < primes.size() && d < 32; ++d) {
    if (primes[d] >= lim) continue;
    double b0 = 3.0;
    for (u64 s : primes)
      if (s < lim) b0 = std::max(b0, std::ceil((double)s / 2.0 / (double)primes[d]));
    if ((b0 + 14.0) * (double)primes[d] < std::ldexp(1.0, 51)) mask |= 1u << d;
  }
  return mask;
}

void build_context(lcl_context* c, size_t degree, int depth, int secure, int device) {
  need(degree >= 8 && (degree & (degree - 1)) == 0, LCL_PARAMETER_ERROR,
       "ring degree must be a power of two >= 8");
  need(degree <= (1u << 17), LCL_PARAMETER_ERROR, "ring degree above 2^17 is not supported");
  need(depth >= 0 && depth + 2 <= LCL_MAXP, LCL_PARAMETER_ERROR, "depth outside supported range");
  int ndev = 0;
  cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  need(device >= 0 && device < ndev, LCL_CUDA_ERROR, "no such CUDA device");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  c->device = device;
  c->n = degree;
  c->logn = __builtin_ctzll(degree);
  c->full = (u32)depth + 1;
  c->scale = std::ldexp(1.0, 40);
  // make_basis (ckks.cpp:77-93): q0 44 bits, depth x 40 bits, special 54 bits.
  std::vector<u64> avoid;
  std::vector<u64> chain = h_ntt_primes(44, degree, 1, avoid);
  avoid.push_back(chain[0]);
  if (depth > 0) {
    for (u64 q : h_ntt_primes(40, degree, depth, avoid)) {
      chain.push_back(q);
      avoid.push_back(q);
    }
  }
  const u64 special = h_ntt_primes(54, degree, 1, avoid)[0];
  if (secure) {
    static const std::map<size_t, double> budget = {
        {1024, 27}, {2048, 54}, {4096, 109}, {8192, 218}, {16384, 438}, {32768, 881},
        {65536, 1770}, {131072, 3540}};
    auto it = budget.find(degree);
    need(it != budget.end(), LCL_PARAMETER_ERROR, "no 128-bit budget entry for this ring degree");
    double total = 0;
    for (u64 q : chain) total += std::log2((double)q);
    total += std::log2((double)special);
    need(total <= it->second, LCL_PARAMETER_ERROR, "modulus chain exceeds the 128-bit budget");
  }
  c->primes = chain;
  c->primes.push_back(special);
  const u32 P = c->P();
  const size_t n = degree;
  std::vector<PrimeConst> pc(P);
  std::vector<ulonglong2> tw(P * n), itw(P * n);
  std::vector<double2> twf(P * n), itwf(P * n);
  for (u32 i = 0; i < P; ++i) {
    const u64 q = c->primes[i];
    const u128 ratio = ~(u128)0 / q;
    PrimeConst& k = pc[i];
    k.q = q;
    k.two_q = 2 * q;
    k.ratio_lo = (u64)ratio;
    k.ratio_hi = (u64)(ratio >> 64);
    k.one_shoup = (u64)(((u128)1 << 64) / q);
    k.half = q >> 1;
    k.n_inv = h_invmod(n, q);
    k.n_inv_shoup = h_shoup(k.n_inv, q);
    // build_tables (rns.cpp:115-138): root[brv(i)] = psi^i, inverse likewise.
    const u64 psi = h_root_2n(n, q), psi_inv = h_invmod(psi, q);
    // iroot[1] = psi^-brv(1) = psi^-(n/2)
    k.w1n = h_mulmod(h_powmod(psi_inv, n / 2, q), k.n_inv, q);
    k.w1n_shoup = h_shoup(k.w1n, q);
    k.mu56 = (u32)(((u128)1 << 56) / q);
    k.mu62 = (u32)(((u128)1 << 62) / q);
    // FP64 companions: every value below 2^53 converts exactly, and w / q is
    // the correctly rounded quotient f_mulmod's error bound assumes
    const double qd = (double)q;
    k.qf = qd;
    k.qinvf = 1.0 / qd;
    k.ninvf = (double)k.n_inv;
    k.ninvq = k.ninvf / qd;
    k.w1nf = (double)k.w1n;
    k.w1nq = k.w1nf / qd;
    u64 f = 1, g = 1;
    for (size_t t = 0; t < n; ++t) {
      const size_t r = h_brv(t, c->logn);
      tw[i * n + r] = make_ulonglong2(f, h_shoup(f, q));
      itw[i * n + r] = make_ulonglong2(g, h_shoup(g, q));
      twf[i * n + r] = make_double2((double)f, (double)f / qd);
      itwf[i * n + r] = make_double2((double)g, (double)g / qd);
      f = h_mulmod(f, psi, q);
      g = h_mulmod(g, psi_inv, q);
    }
  }
  std::vector<u64> smod(P * P);
  std::vector<ulonglong2> pinv(P * P);
  for (u32 s = 0; s < P; ++s)
    for (u32 d = 0; d < P; ++d) {
      smod[s * P + d] = c->primes[s] % c->primes[d];
      const u64 iv = s == d ? 0 : h_invmod(c->primes[s], c->primes[d]);
      pinv[s * P + d] = make_ulonglong2(iv, h_shoup(iv, c->primes[d]));
    }
  cuda_check(cudaMalloc(&c->d_primes, P * sizeof(PrimeConst)), "alloc");
  cuda_check(cudaMalloc(&c->d_tw, P * n * sizeof(ulonglong2)), "alloc");
  cuda_check(cudaMalloc(&c->d_itw, P * n * sizeof(ulonglong2)), "alloc");
  cuda_check(cudaMalloc(&c->d_twf, P * n * sizeof(double2)), "alloc");
  cuda_check(cudaMalloc(&c->d_itwf, P * n * sizeof(double2)), "alloc");
  cuda_check(cudaMalloc(&c->d_smod, P * P * 8), "alloc");
  cuda_check(cudaMalloc(&c->d_pinv, P * P * sizeof(ulonglong2)), "alloc");
  cuda_check(cudaMemcpy(c->d_primes, pc.data(), P * sizeof(PrimeConst), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_tw, tw.data(), P * n * sizeof(ulonglong2), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_itw, itw.data(), P * n * sizeof(ulonglong2), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_twf, twf.data(), P * n * sizeof(double2), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_itwf, itwf.data(), P * n * sizeof(double2), cudaMemcpyHostToDevice), "upload");
  if (c->logn >= 13) {
    // block-ordered tables: block b (N1 = n / 256 blocks) holds
    // root[(N1 + b) 2^lm + i] at blk_tw_pos(lm, i mod 2^(lm-4), i div 2^(lm-4))
    // (lm >= 4), 2^lm - 1 + i (lm < 4); entry 255 of each block is unused
    const size_t n1 = n >> 8;
    std::vector<ulonglong2> btw(P * n, make_ulonglong2(0, 0)), bitw(P * n, make_ulonglong2(0, 0));
    std::vector<double2> btwf(P * n, make_double2(0, 0)), bitwf(P * n, make_double2(0, 0));
    for (u32 i = 0; i < P; ++i)
      for (size_t b = 0; b < n1; ++b)
        for (int lm = 0; lm < 8; ++lm)
          for (u32 x = 0; x < (1u << lm); ++x) {
            const u32 pos = lm < 4 ? blk_tw_pos(lm, x, 0) : blk_tw_pos(lm, x & ((1u << (lm - 4)) - 1), x >> (lm - 4));
            const size_t src = i * n + (n1 + b) * ((size_t)1 << lm) + x, dst = i * n + b * 256 + pos;
            btw[dst] = tw[src];
            bitw[dst] = itw[src];
            btwf[dst] = twf[src];
            bitwf[dst] = itwf[src];
          }
    cuda_check(cudaMalloc(&c->d_btw, P * n * sizeof(ulonglong2)), "alloc");
    cuda_check(cudaMalloc(&c->d_bitw, P * n * sizeof(ulonglong2)), "alloc");
    cuda_check(cudaMalloc(&c->d_btwf, P * n * sizeof(double2)), "alloc");
    cuda_check(cudaMalloc(&c->d_bitwf, P * n * sizeof(double2)), "alloc");
    cuda_check(cudaMemcpy(c->d_btw, btw.data(), P * n * sizeof(ulonglong2), cudaMemcpyHostToDevice), "upload");
    cuda_check(cudaMemcpy(c->d_bitw, bitw.data(), P * n * sizeof(ulonglong2), cudaMemcpyHostToDevice), "upload");
    cuda_check(cudaMemcpy(c->d_btwf, btwf.data(), P * n * sizeof(double2), cudaMemcpyHostToDevice), "upload");
    cuda_check(cudaMemcpy(c->d_bitwf, bitwf.data(), P * n * sizeof(double2), cudaMemcpyHostToDevice), "upload");
  }
  c->fp_mask = fp_rows(c->primes);
  {
    // pair_accumulate_f64 needs |x - y| < 2^44 for every q-chain residue
    const char* env = std::getenv("LCL_PAIR_F64");
    bool ok = !(env && env[0] == '0');
    for (u32 d = 0; d < c->full; ++d) ok = ok && c->primes[d] < (1ull << 44);
    c->pair_f64 = ok;
  }
  cuda_check(cudaMemcpy(c->d_smod, smod.data(), P * P * 8, cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(c->d_pinv, pinv.data(), P * P * sizeof(ulonglong2), cudaMemcpyHostToDevice), "upload");
}

void free_context(lcl_context* c) {
  for (auto& ln : c->lanes) {
    for (DevBuf* b : {&ln.ws_coef, &ln.ws_digits, &ln.ws_acc, &ln.ws_coefsp, &ln.ws_mid,
                      &ln.ws_tern, &ln.ws_ctA, &ln.ws_ctB, &ln.ws_ctC, &ln.ws_c1inv})
      b->release();
    if (ln.done) cudaEventDestroy(ln.done);
    if (ln.stream) cudaStreamDestroy(ln.stream);
  }
  c->lanes.clear();
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  c->fork_ev = nullptr;
  cudaFree(c->d_primes);
  cudaFree(c->d_tw);
  cudaFree(c->d_itw);
  cudaFree(c->d_twf);
  cudaFree(c->d_itwf);
  cudaFree(c->d_btw);
  cudaFree(c->d_bitw);
  cudaFree(c->d_btwf);
  cudaFree(c->d_bitwf);
  cudaFree(c->d_smod);
  cudaFree(c->d_pinv);
  cudaFree(c->d_pairs);
  for (auto& kv : c->sched) cudaFree(kv.second);
  if (c->unpk) cudaStreamDestroy(c->unpk);
  if (c->d2h_agg) cudaStreamDestroy(c->d2h_agg);
  if (c->crit) cudaStreamDestroy(c->crit);
  if (c->crit2) cudaStreamDestroy(c->crit2);
  if (c->lo) cudaStreamDestroy(c->lo);
  if (c->crit3) cudaStreamDestroy(c->crit3);
  for (cudaEvent_t e : c->unpk_ev) cudaEventDestroy(e);
  cudaFree(c->d_relin);
  cudaFree(c->d_relin_shoup);
  for (auto& kv : c->d_rot) cudaFree(kv.second);
  for (auto& kv : c->d_rot_shoup) cudaFree(kv.second);
  for (auto& kv : c->d_perm) cudaFree(kv.second);
  for (auto& kv : c->d_blkmap) cudaFree(kv.second);
  for (auto& kv : c->d_sigma) cudaFree(kv.second);
  for (DevBuf* b : {&c->ws_coef, &c->ws_digits, &c->ws_acc, &c->ws_coefsp, &c->ws_mid,
                    &c->ws_tern, &c->ws_ctA, &c->ws_ctB, &c->ws_ctC, &c->ws_pt, &c->ws_c1inv, &c->ws_io_in,
                    &c->ws_io_sel, &c->ws_io_dist, &c->ws_io_agg, &c->ws_dtern, &c->ws_atern,
                    &c->ws_ptl, &c->ws_rows, &c->ws_cal, &c->ws_stage, &c->ws_stage_sel,
                    &c->ws_err, &c->ws_slots,
                    &c->ws_enc, &c->ws_enc_in})
    b->release();
  for (void* p : {(void*)c->d_twist, (void*)c->d_roots, (void*)c->d_brv, (void*)c->d_slot})
    if (p) cudaFree(p);
  c->d_twist = c->d_roots = nullptr;
  c->d_brv = c->d_slot = nullptr;
  c->ws_dec.release();
  for (cudaEvent_t e : c->io_ev) cudaEventDestroy(e);
  c->io_ev.clear();
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  c->h2d = c->d2h = nullptr;
}

u64 key_words(const lcl_context* c) { return (u64)c->full * 2 * c->P() * c->N(); }

u64* upload_key(lcl_context* c, const u64* h, size_t words, u64** shoup_out) {
  need(h != nullptr, LCL_KEY_ERROR, "null key");
  need(words == key_words(c), LCL_KEY_ERROR, "switch key has the wrong shape");
  // Companions for the fused inner product: Shoup floor(k * 2^64 / q_row) on
  // integer rows, the key word as a double on FP64 rows.
  std::vector<u64> sh(words);
  const u64 N = c->N();
  const u32 P = c->P();
  for (size_t i = 0; i < words; ++i) {
    const u32 row = (u32)((i / N) % P);
    const u64 q = c->primes[row];
    need(h[i] < q, LCL_KEY_ERROR, "key residue outside its modulus");
    if ((c->fp_mask >> row) & 1u) {
      const double kd = (double)h[i];  // FP64 rows: the key word as a double
      std::memcpy(&sh[i], &kd, 8);
    } else {
      sh[i] = h_shoup(h[i], q);
    }
  }
  u64* d = nullptr;
  u64* ds = nullptr;
  cuda_check(cudaMalloc(&d, words * 8), "key alloc");
  cuda_check(cudaMalloc(&ds, words * 8), "key alloc");
  cuda_check(cudaMemcpy(d, h, words * 8, cudaMemcpyHostToDevice), "key upload");
  cuda_check(cudaMemcpy(ds, sh.data(), words * 8, cudaMemcpyHostToDevice), "key upload");
  *shoup_out = ds;
  return d;
}

// galois_elt_for_rotation + make_galois_tables (rns.cpp:508-532).
std::vector<u32> galois_perm(size_t n, int logn, size_t step) {
  const u64 two_n = 2 * (u64)n;
  u64 elt = 1;
  for (size_t i = 0; i < step % (n / 2); ++i) elt = (elt * 5) % two_n;
  std::vector<u32> p(n);
  for (size_t i = 0; i < n; ++i) {
    const u64 e = 2 * (u64)h_brv(i, logn) + 1;
    const u64 t = (e * elt) % two_n;
    p[i] = (u32)h_brv((size_t)((t - 1) / 2), logn);
  }
  return p;
}

// The same automorphism on coefficients: y(X) = x(X^elt), gathered as
// y[k] = +-x[src] with src = k * elt^-1 mod 2N folded into [0, N).
std::vector<u32> galois_sigma(size_t n, size_t step) {
  const u64 two_n = 2 * (u64)n;
  u64 elt = 1;
  for (size_t i = 0; i < step % (n / 2); ++i) elt = (elt * 5) % two_n;
  // elt is odd, so it is invertible mod 2N (a power of two): Newton iteration
  u64 inv = elt;
  for (int i = 0; i < 6; ++i) inv = (inv * (2 - elt * inv)) % two_n;
  inv %= two_n;
  std::vector<u32> s(n);
  for (size_t k = 0; k < n; ++k) {
    const u64 src = ((u64)k * inv) % two_n;
    s[k] = src < n ? (u32)src : ((u32)(src - n) | 0x80000000u);
  }
  return s;
}

void check_count(const lcl_context* c, size_t count) {
  need(count >= 1 && count <= c->full, LCL_BASIS_MISMATCH, "prime count outside the basis");
}

}  // namespace

extern "C" {

const char* lcl_last_error(void) { return g_last_error.c_str(); }

int lcl_context_create(size_t degree, int depth, int secure, int device, lcl_context** out) {
  return guarded([&] {
    need(out != nullptr, LCL_USAGE_ERROR, "null output handle");
    auto c = std::make_unique<lcl_context>();
    try {
      build_context(c.get(), degree, depth, secure, device);
    } catch (...) {
      free_context(c.get());
      throw;
    }
    *out = c.release();
  });
}

int lcl_context_destroy(lcl_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    free_context(ctx);
    delete ctx;
  });
}

int lcl_context_primes(const lcl_context* ctx, uint64_t* primes, size_t* full) {
  return guarded([&] {
    if (full) *full = ctx->full;
    if (primes) std::copy(ctx->primes.begin(), ctx->primes.end(), primes);
  });
}

int lcl_set_stream(lcl_context* ctx, void* s) {
  return guarded([&] { ctx->stream = static_cast<cudaStream_t>(s); });
}

int lcl_synchronize(lcl_context* ctx) {
  return guarded([&] { cuda_check(cudaStreamSynchronize(ctx->stream), "synchronize"); });
}

int lcl_get_counts(const lcl_context* ctx, lcl_counts* out) {
  return guarded([&] { *out = ctx->counts; });
}

int lcl_reset_counts(lcl_context* ctx) {
  return guarded([&] { ctx->counts = lcl_counts{}; });
}

uint64_t lcl_launch_count(const lcl_context* ctx) { return ctx ? ctx->launches : 0; }

int lcl_peak_butterflies(lcl_context* ctx, double* gbfly_per_s) {
  return guarded([&] {
    const u32 blocks = 148 * 8, threads = 256, iters = 4096;
    u64* sink = ctx->ws_pt.get((u64)blocks * threads);
    const u64 q = ctx->primes[0];
    const u64 w = q / 3 + 7;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    lcl::peak_butterfly<<<blocks, threads, 0, ctx->stream>>>(sink, 64, q, w, h_shoup(w, q));
    cudaEventRecord(a, ctx->stream);
    lcl::peak_butterfly<<<blocks, threads, 0, ctx->stream>>>(sink, iters, q, w, h_shoup(w, q));
    cudaEventRecord(b, ctx->stream);
    cuda_check(cudaEventSynchronize(b), "peak butterfly");
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *gbfly_per_s = (double)blocks * threads * iters * 16 / (ms * 1e-3) / 1e9;
  });
}

int lcl_peak_butterflies_f64(lcl_context* ctx, double* gbfly_per_s) {
  return guarded([&] {
    const u32 blocks = 148 * 8, threads = 256, iters = 4096;
    u64* sink = ctx->ws_pt.get((u64)blocks * threads);
    const double q = (double)ctx->primes[1], w = std::floor(q / 3) + 7, wq = w / q;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    lcl::peak_butterfly_f64<<<blocks, threads, 0, ctx->stream>>>(sink, 64, q, w, wq);
    cudaEventRecord(a, ctx->stream);
    lcl::peak_butterfly_f64<<<blocks, threads, 0, ctx->stream>>>(sink, iters, q, w, wq);
    cudaEventRecord(b, ctx->stream);
    cuda_check(cudaEventSynchronize(b), "peak butterfly f64");
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *gbfly_per_s = (double)blocks * threads * iters * 16 / (ms * 1e-3) / 1e9;
  });
}

int lcl_profile_begin(lcl_context* ctx) {
  return guarded([&] {
    for (auto& r : ctx->prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    ctx->prof.clear();
    ctx->prof_on = true;
  });
}

int lcl_profile_end(lcl_context* ctx, char* json, size_t cap) {
  return guarded([&] {
    ctx->prof_on = false;
    cuda_check(cudaStreamSynchronize(ctx->stream), "profile sync");
    struct Agg {
      double ms = 0, bytes = 0, bfly = 0;
      u64 launches = 0;
    };
    std::map<std::string, Agg> agg;
    for (auto& r : ctx->prof) {
      float ms = 0;
      cudaEventElapsedTime(&ms, r.a, r.b);
      Agg& a = agg[r.name];
      a.ms += ms;
      a.bytes += r.bytes;
      a.bfly += r.bfly;
      a.launches += 1;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    ctx->prof.clear();
    std::string s = "[";
    bool first = true;
    for (auto& kv : agg) {
      char buf[256];
      std::snprintf(buf, sizeof buf,
                    "%s{\"name\": \"%s\", \"launches\": %llu, \"ms\": %.6f, \"bytes\": %.0f, "
                    "\"bfly\": %.0f}",
                    first ? "" : ", ", kv.first.c_str(), (unsigned long long)kv.second.launches,
                    kv.second.ms, kv.second.bytes, kv.second.bfly);
      s += buf;
      first = false;
    }
    s += "]";
    need(s.size() + 1 <= cap, LCL_USAGE_ERROR, "profile buffer too small");
    std::memcpy(json, s.c_str(), s.size() + 1);
  });
}

int lcl_upload_relin_key(lcl_context* ctx, const uint64_t* h_key, size_t words) {
  return guarded([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    u64* ds = nullptr;
    u64* d = upload_key(ctx, h_key, words, &ds);
    if (ctx->d_relin) cudaFree(ctx->d_relin);
    if (ctx->d_relin_shoup) cudaFree(ctx->d_relin_shoup);
    ctx->d_relin = d;
    ctx->d_relin_shoup = ds;
  });
}

int lcl_upload_rotation_key(lcl_context* ctx, size_t step, const uint64_t* h_key, size_t words) {
  return guarded([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    step %= ctx->n / 2;
    need(step != 0, LCL_KEY_ERROR, "rotation step 0 needs no key");
    u64* ds = nullptr;
    u64* d = upload_key(ctx, h_key, words, &ds);
    auto it = ctx->d_rot.find(step);
    if (it != ctx->d_rot.end()) {
      cudaFree(it->second);
      cudaFree(ctx->d_rot_shoup[step]);
    }
    ctx->d_rot[step] = d;
    ctx->d_rot_shoup[step] = ds;
    if (!ctx->d_perm.count(step)) {
      const std::vector<u32> p = galois_perm(ctx->n, ctx->logn, step);
      u32* dp = nullptr;
      cuda_check(cudaMalloc(&dp, p.size() * 4), "perm alloc");
      cuda_check(cudaMemcpy(dp, p.data(), p.size() * 4, cudaMemcpyHostToDevice), "perm upload");
      ctx->d_perm[step] = dp;
      if (ctx->logn >= 13) {
        // the evaluation-domain permutation is block-local (block_gather):
        // output block b reads only source block p[256 b] >> 8
        const size_t nb = ctx->n >> 8;
        std::vector<u32> bm(nb, 0xFFFFFFFFu);
        for (size_t b = 0; b < nb; ++b) bm[p[b << 8] >> 8] = (u32)b;
        for (u32 v : bm) need(v != 0xFFFFFFFFu, LCL_PARAMETER_ERROR, "Galois permutation is not block-local");
        u32* db = nullptr;
        cuda_check(cudaMalloc(&db, nb * 4), "blkmap alloc");
        cuda_check(cudaMemcpy(db, bm.data(), nb * 4, cudaMemcpyHostToDevice), "blkmap upload");
        ctx->d_blkmap[step] = db;
      }
      const std::vector<u32> sg = galois_sigma(ctx->n, step);
      u32* ds = nullptr;
      cuda_check(cudaMalloc(&ds, sg.size() * 4), "sigma alloc");
      cuda_check(cudaMemcpy(ds, sg.data(), sg.size() * 4, cudaMemcpyHostToDevice), "sigma upload");
      ctx->d_sigma[step] = ds;
    }
  });
}

int lcl_has_rotation_key(const lcl_context* ctx, size_t step) {
  return ctx->d_rot.count(step % (ctx->n / 2)) ? 1 : 0;
}

int lcl_device_alloc(lcl_context* ctx, size_t bytes, void** d_ptr) {
  return guarded([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_check(cudaMalloc(d_ptr, bytes), "cudaMalloc");
  });
}

int lcl_device_free(lcl_context* ctx, void* d_ptr) {
  return guarded([&] { cuda_check(cudaFree(d_ptr), "cudaFree"); (void)ctx; });
}

int lcl_copy_h2d(lcl_context* ctx, void* d_dst, const void* h_src, size_t bytes) {
  return guarded([&] {
    cuda_check(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, ctx->stream), "h2d");
    cuda_check(cudaStreamSynchronize(ctx->stream), "h2d sync");
  });
}

int lcl_copy_d2h(lcl_context* ctx, void* h_dst, const void* d_src, size_t bytes) {
  return guarded([&] {
    cuda_check(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    cuda_check(cudaStreamSynchronize(ctx->stream), "d2h sync");
  });
}

static int ntt_common(lcl_context* ctx, uint64_t* d, size_t items, size_t count, int sp, bool inv) {
  return guarded([&] {
    check_count(ctx, count);
    const u32 rpi = (u32)count + (sp ? 1 : 0);
    std::vector<u32> p(rpi);
    for (u32 i = 0; i < rpi; ++i) p[i] = i < count ? i : ctx->full;
    const RowMap m = make_map(d, rpi, ctx->N(), (u64)rpi * ctx->N(), 1, 0, p);
    const u32 rows = (u32)(items * rpi);
    if (inv)
      launch_inv(ctx, rows, m, PlainStore{m});
    else
      launch_fwd(ctx, rows, m, PlainLoad{m}, PlainStore{m});
  });
}

int lcl_ntt_forward(lcl_context* ctx, uint64_t* d, size_t items, size_t count, int sp) {
  return ntt_common(ctx, d, items, count, sp, false);
}
int lcl_ntt_inverse(lcl_context* ctx, uint64_t* d, size_t items, size_t count, int sp) {
  return ntt_common(ctx, d, items, count, sp, true);
}

static int addsub(lcl_context* ctx, const uint64_t* a, const uint64_t* b, size_t batch,
                  size_t count, uint64_t* out, bool sub) {
  return guarded([&] {
    check_count(ctx, count);
    const u32 m = (u32)count;
    const u64 N = ctx->N();
    const RowMap o = ct_map(out, m, N, 2ull * m * N), x = ct_map(a, m, N, 2ull * m * N),
                 y = ct_map(b, m, N, 2ull * m * N);
    const u32 rows = (u32)(batch * 2 * m);
    const u32 grid = (u32)(((u64)rows * N + 255) / 256);
    if (sub)
      rows_addsub<true><<<grid, 256, 0, ctx->stream>>>(o, x, y, rows, ctx->logn, ctx->d_primes);
    else
      rows_addsub<false><<<grid, 256, 0, ctx->stream>>>(o, x, y, rows, ctx->logn, ctx->d_primes);
    post_launch(ctx);
    ctx->counts.additions += batch;
  });
}

int lcl_hadd(lcl_context* ctx, const uint64_t* a, const uint64_t* b, size_t batch, size_t count,
             uint64_t* out) {
  return addsub(ctx, a, b, batch, count, out, false);
}
int lcl_hsub(lcl_context* ctx, const uint64_t* a, const uint64_t* b, size_t batch, size_t count,
             uint64_t* out) {
  return addsub(ctx, a, b, batch, count, out, true);
}

int lcl_hmult(lcl_context* ctx, const uint64_t* d_a, const uint64_t* d_b, size_t batch,
              size_t count, uint64_t* d_tern) {
  return guarded([&] {
    check_count(ctx, count);
    const u64 total = (u64)batch * count * ctx->N();
    if (total == 0) return;
    ProfScope ps(ctx, "ct_tensor", 8.0 * (double)total * (d_a == d_b ? 5 : 7));
    ct_tensor<<<(u32)((total + 255) / 256), 256, 0, ctx->stream>>>(
        d_a, d_b, (u32)batch, (u32)count, ctx->logn, d_tern, ctx->d_primes);
    post_launch(ctx);
    ctx->counts.multiplications += batch;
  });
}

int lcl_hsquare(lcl_context* ctx, const uint64_t* d_a, size_t batch, size_t count,
                uint64_t* d_tern) {
  return lcl_hmult(ctx, d_a, d_a, batch, count, d_tern);
}

int lcl_relinearize(lcl_context* ctx, const uint64_t* d_tern, size_t batch, size_t count,
                    uint64_t* d_out) {
  return guarded([&] {
    check_count(ctx, count);
    relinearize_batch(ctx, d_tern, (u32)batch, (u32)count, d_out);
  });
}

int lcl_rescale(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                uint64_t* d_out) {
  return guarded([&] {
    check_count(ctx, count);
    rescale_batch(ctx, d_ct, (u32)batch, (u32)count, d_out);
  });
}

int lcl_rotate(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count, size_t step,
               uint64_t* d_out) {
  return guarded([&] {
    check_count(ctx, count);
    step = norm_step(ctx, step);
    const u64 words = (u64)batch * 2 * count * ctx->N();
    if (step == 0) {
      cuda_check(cudaMemcpyAsync(d_out, d_ct, words * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
      return;
    }
    rotate_level(ctx, d_ct, (u32)batch, (u32)count, step, d_out, false);
  });
}

int lcl_hoisted_rotations(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                          const size_t* h_steps, size_t nsteps, uint64_t* d_outs) {
  return guarded([&] {
    check_count(ctx, count);
    hoisted_batch(ctx, d_ct, (u32)batch, (u32)count, h_steps, nsteps, d_outs);
  });
}

int lcl_calibrate(lcl_context* ctx, const uint64_t* d_ct, size_t count, double* t_hoist,
                  double* t_decompose, double* m_cipher) {
  return guarded([&] {
    check_count(ctx, count);
    need(lcl_has_rotation_key(ctx, 1) && lcl_has_rotation_key(ctx, 2), LCL_KEY_ERROR,
         "calibration needs rotation keys for steps 1 and 2");
    const u32 m = (u32)count;
    const u64 words = 2ull * m * ctx->N();
    u64* outs = ctx->ws_cal.get(2 * words);
    cudaEvent_t a, b;
    cuda_check(cudaEventCreate(&a), "event");
    cuda_check(cudaEventCreate(&b), "event");
    // median of 11 device-timed calls (protocol.cpp:232-243)
    auto median_time = [&](const std::vector<size_t>& steps) {
      std::vector<double> t;
      for (int rep = 0; rep < 11; ++rep) {
        cuda_check(cudaEventRecord(a, ctx->stream), "record");
        hoisted_batch(ctx, d_ct, 1, m, steps.data(), steps.size(), outs);
        cuda_check(cudaEventRecord(b, ctx->stream), "record");
        cuda_check(cudaEventSynchronize(b), "sync");
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
        t.push_back(ms * 1e-3);
      }
      std::sort(t.begin(), t.end());
      return t[t.size() / 2];
    };
    const double t1 = median_time({1});
    const double t2 = median_time({1, 2});
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    // the reference's naming (protocol.cpp:249-250): t_hoist = decompose +
    // first rotation, t_decompose = the marginal hoisted rotation
    if (t_hoist) *t_hoist = std::max(t1, 1e-9);
    if (t_decompose) *t_decompose = std::max(t2 - t1, 1e-9);
    if (m_cipher) *m_cipher = (double)(words * 8);  // Ciphertext::size_bytes
  });
}

int lcl_slot_reduce(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                    size_t width, size_t k, uint64_t* d_out) {
  return guarded([&] {
    check_count(ctx, count);
    slot_reduce_batch(ctx, d_ct, (u32)batch, (u32)count, width, k, d_out);
  });
}

int lcl_mult_plain_const(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                         double value, double pt_scale, uint64_t* d_out) {
  return guarded([&] {
    check_count(ctx, count);
    const u32 m = (u32)count;
    const u64 N = ctx->N();
    std::vector<double> v(ctx->n / 2, value);
    const std::vector<long long> rounded = h_encode_rounded(v, ctx->n, pt_scale);
    std::vector<u64> pt((u64)m * N);
    for (u32 r = 0; r < m; ++r) {
      const u64 q = ctx->primes[r];
      for (u64 i = 0; i < N; ++i) {
        const long long x = rounded[i];
        const u64 mag = (u64)(x < 0 ? -x : x) % q;
        pt[r * N + i] = x < 0 ? (mag == 0 ? 0 : q - mag) : mag;
      }
    }
    u64* d_pt = ctx->ws_pt.get(pt.size());
    cuda_check(cudaMemcpyAsync(d_pt, pt.data(), pt.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "pt");
    const RowMap ptm = make_map(d_pt, m, N, (u64)m * N, 1, 0, ctx->primes_0(m));
    launch_fwd(ctx, m, ptm, PlainLoad{ptm}, PlainStore{ptm});
    const u64 total = (u64)batch * 2 * m * N;
    mult_plain<<<(u32)((total + 255) / 256), 256, 0, ctx->stream>>>(d_ct, d_pt, (u32)batch, m,
                                                                    ctx->logn, d_out, ctx->d_primes);
    post_launch(ctx);
    cuda_check(cudaStreamSynchronize(ctx->stream), "mult_plain");
    ctx->counts.multiplications += batch;
  });
}

uint64_t lcl_derive_seed(uint64_t root, uint64_t tag) {  // sampling.cpp:24-30
  u64 z = root + 0x9e3779b97f4a7c15ull * (tag + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int lcl_sampler_create(uint64_t seed, lcl_sampler** out) {
  return guarded([&] {
    need(out != nullptr, LCL_PARAMETER_ERROR, "null output");
    *out = new lcl_sampler(seed);
  });
}

int lcl_sampler_destroy(lcl_sampler* s) {
  delete s;
  return LCL_OK;
}

int lcl_sampler_uniform_real(lcl_sampler* s, size_t count, double* out) {
  return guarded([&] {
    for (size_t i = 0; i < count; ++i) out[i] = s->uniform_real();
  });
}

int lcl_pack_and_encrypt(lcl_context* ctx, lcl_sampler* rng, const double* h_weights,
                         size_t dim, double prescale, const uint64_t* d_pk, uint64_t* d_out) {
  return guarded([&] {
    need(rng != nullptr && d_pk != nullptr, LCL_PARAMETER_ERROR, "null sampler or key");
    pack_and_encrypt(ctx, rng, h_weights, dim, prescale, d_pk, d_out);
  });
}

int lcl_generate_keys(lcl_context* ctx, lcl_sampler* rng, const size_t* steps, size_t nsteps,
                      uint64_t* d_sk, uint64_t* d_pk, uint64_t* d_relin, uint64_t* d_rot,
                      size_t* rot_steps, size_t* n_rot) {
  return guarded([&] {
    need(rng != nullptr, LCL_PARAMETER_ERROR, "null sampler");
    const size_t k = generate_keys(ctx, rng, steps, nsteps, d_sk, d_pk, d_relin, d_rot, rot_steps);
    if (n_rot) *n_rot = k;
  });
}

int lcl_build_mask(lcl_context* ctx, lcl_sampler* rng, size_t n, const size_t* selected,
                   size_t l, const uint64_t* d_pk, uint64_t* d_rank_rows, uint64_t* d_selectors) {
  return guarded([&] {
    need(rng != nullptr && d_pk != nullptr, LCL_PARAMETER_ERROR, "null sampler or key");
    build_mask(ctx, rng, n, selected, l, d_pk, d_rank_rows, d_selectors);
  });
}

int lcl_decrypt(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                const uint64_t* d_sk, uint64_t* d_pt) {
  return guarded([&] {
    check_count(ctx, count);
    need(d_sk != nullptr, LCL_KEY_ERROR, "null secret key");
    decrypt_batch(ctx, d_ct, (u32)batch, (u32)count, d_sk, d_pt);
  });
}

int lcl_decode(lcl_context* ctx, uint64_t* d_pt, size_t batch, size_t count, double scale,
               double* d_slots) {
  return guarded([&] {
    check_count(ctx, count);
    decode_batch(ctx, d_pt, (u32)batch, (u32)count, scale, d_slots);
  });
}

int lcl_decrypt_values(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                       double scale, const uint64_t* d_sk, double* d_slots) {
  return guarded([&] {
    check_count(ctx, count);
    need(d_sk != nullptr, LCL_KEY_ERROR, "null secret key");
    u64* pt = ctx->ws_pt.get((u64)batch * count * ctx->N());
    decrypt_batch(ctx, d_ct, (u32)batch, (u32)count, d_sk, pt);
    decode_batch(ctx, pt, (u32)batch, (u32)count, scale, d_slots);
  });
}

// table_from_matrix / totals_from_matrix (aggregation.cpp:242-277) on the
// device: decrypt_values of every entry, entry_values, then the host fills
// the symmetric table (per_pair) or the totals (row_sums) in the reference's
// order.
static void entry_values_batch(lcl_context* ctx, const uint64_t* d_entries, size_t entries,
                               size_t count, double scale, int reduced, double value_scale,
                               const uint64_t* d_sk, std::vector<double>& vals) {
  check_count(ctx, count);
  need(d_sk != nullptr, LCL_KEY_ERROR, "null secret key");
  need(value_scale != 0.0, LCL_PARAMETER_ERROR, "zero value scale");
  vals.assign(entries, 0.0);
  if (!entries) return;
  const u32 h = (u32)(ctx->n / 2);
  u64* pt = ctx->ws_pt.get((u64)entries * count * ctx->N());
  double* slots = reinterpret_cast<double*>(ctx->ws_slots.get((u64)entries * h + entries));
  double* dv = slots + (u64)entries * h;
  decrypt_batch(ctx, d_entries, (u32)entries, (u32)count, d_sk, pt);
  decode_batch(ctx, pt, (u32)entries, (u32)count, scale, slots);
  entry_values<<<(u32)((entries + 127) / 128), 128, 0, ctx->stream>>>(
      slots, (u32)entries, h, reduced, value_scale, dv);
  post_launch(ctx);
  cuda_check(cudaMemcpyAsync(vals.data(), dv, entries * 8, cudaMemcpyDeviceToHost, ctx->stream),
             "d2h values");
  cuda_check(cudaStreamSynchronize(ctx->stream), "values sync");
}

int lcl_table_from_matrix(lcl_context* ctx, const uint64_t* d_entries, size_t n, size_t count,
                          double scale, int reduced, double value_scale, const uint64_t* d_sk,
                          double* h_table) {
  return guarded([&] {
    std::vector<double> v;
    entry_values_batch(ctx, d_entries, n * (n - 1) / 2, count, scale, reduced, value_scale, d_sk, v);
    for (size_t i = 0; i < n * n; ++i) h_table[i] = 0.0;
    size_t p = 0;
    for (size_t i = 0; i < n; ++i)
      for (size_t j = i + 1; j < n; ++j, ++p) h_table[i * n + j] = h_table[j * n + i] = v[p];
  });
}

int lcl_totals_from_matrix(lcl_context* ctx, const uint64_t* d_entries, size_t n, int mode,
                           size_t count, double scale, int reduced, double value_scale,
                           const uint64_t* d_sk, double* h_totals) {
  return guarded([&] {
    need(mode == LCL_PER_PAIR || mode == LCL_ROW_SUMS, LCL_USAGE_ERROR, "unknown distance mode");
    std::vector<double> v;
    if (mode == LCL_ROW_SUMS) {
      entry_values_batch(ctx, d_entries, n, count, scale, reduced, value_scale, d_sk, v);
      for (size_t i = 0; i < n; ++i) h_totals[i] = v[i];
      return;
    }
    entry_values_batch(ctx, d_entries, n * (n - 1) / 2, count, scale, reduced, value_scale, d_sk, v);
    std::vector<double> t(n * n, 0.0);
    size_t p = 0;
    for (size_t i = 0; i < n; ++i)
      for (size_t j = i + 1; j < n; ++j, ++p) t[i * n + j] = t[j * n + i] = v[p];
    for (size_t i = 0; i < n; ++i) {  // std::accumulate over the row, left to right
      double a = 0.0;
      for (size_t j = 0; j < n; ++j) a += t[i * n + j];
      h_totals[i] = a;
    }
  });
}

int lcl_pairwise_distance(lcl_context* ctx, const uint64_t* d_a, const uint64_t* d_b,
                          size_t chunks, int lazy, uint64_t* d_out) {
  return guarded([&] {
    // Two "clients" laid out as [2][chunks][...] are required by the pair
    // kernel; stage them contiguously.
    const u32 m = ctx->full;
    const u64 ctw = 2ull * m * ctx->N();
    u64* both = ctx->ws_io_in.get(2 * chunks * ctw);
    cuda_check(cudaMemcpyAsync(both, d_a, chunks * ctw * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    cuda_check(cudaMemcpyAsync(both + chunks * ctw, d_b, chunks * ctw * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    distance_matrix(ctx, both, 2, (u32)chunks, 1, 1, lazy != 0, false, d_out);
  });
}

int lcl_distance_matrix(lcl_context* ctx, const uint64_t* d_clients, size_t n, size_t chunks,
                        double in_scale, size_t width, size_t k, int lazy, int reduce,
                        uint64_t* d_out, double* out_scale) {
  return guarded([&] {
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    distance_matrix(ctx, d_clients, (u32)n, (u32)chunks, width, k, lazy != 0, reduce != 0, d_out);
    if (out_scale) *out_scale = (in_scale * in_scale) / (double)ctx->primes[ctx->full - 1];
  });
}

int lcl_build_distance_matrix(lcl_context* ctx, const uint64_t* d_clients, size_t n,
                              size_t chunks, double in_scale, size_t width, size_t k, int mode,
                              int lazy, int reduce_on_server, uint64_t* d_out, double* out_scale) {
  return guarded([&] {
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    need(mode == LCL_PER_PAIR || mode == LCL_ROW_SUMS, LCL_USAGE_ERROR, "unknown distance mode");
    if (mode == LCL_PER_PAIR)
      distance_matrix(ctx, d_clients, (u32)n, (u32)chunks, width, k, lazy != 0,
                      reduce_on_server != 0, d_out);
    else
      distance_rows(ctx, d_clients, (u32)n, (u32)chunks, width, k, lazy != 0,
                    reduce_on_server != 0, d_out);
    if (out_scale) *out_scale = (in_scale * in_scale) / (double)ctx->primes[ctx->full - 1];
  });
}

int lcl_distance_matrix_pairs(lcl_context* ctx, const uint64_t* d_clients, size_t n,
                              size_t chunks, double in_scale, size_t width, size_t k, int lazy,
                              int reduce, size_t pair_begin, size_t pair_end, uint64_t* d_out,
                              double* out_scale) {
  return guarded([&] {
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    need(pair_begin <= pair_end && pair_end <= n * (n - 1) / 2, LCL_SHAPE_ERROR,
         "pair range outside the matrix");
    if (pair_end > pair_begin)
      distance_matrix(ctx, d_clients, (u32)n, (u32)chunks, width, k, lazy != 0, reduce != 0, d_out,
                      (u32)pair_begin, (u32)pair_end);
    if (out_scale) *out_scale = (in_scale * in_scale) / (double)ctx->primes[ctx->full - 1];
  });
}

int lcl_pair_partials(lcl_context* ctx, const uint64_t* d_clients, size_t n, size_t chunks,
                      uint64_t* d_tern) {
  return guarded([&] {
    need(n >= 2 && n <= 65535, LCL_SHAPE_ERROR, "pairwise distances need 2..65535 clients");
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    const u32 P = (u32)(n * (n - 1) / 2);
    ensure_pairs(ctx, (u32)n);
    pair_accumulate_launch(ctx, d_clients, (u32)n, (u32)chunks, 0, (u32)chunks, row_range(0, P),
                           d_tern, false);
    ctx->counts.multiplications += (u64)P * chunks;
    ctx->counts.additions += (u64)P * (2ull * chunks - 1);
  });
}

int lcl_pair_combine(lcl_context* ctx, uint64_t* d_tern, size_t pairs, size_t shards) {
  return guarded([&] {
    need(shards >= 1 && shards <= 4096, LCL_PARAMETER_ERROR, "shard count outside 1..4096");
    const u32 m = ctx->full;
    const u64 words = (u64)pairs * 3 * m * ctx->N();
    if (words) {
      ProfScope ps(ctx, "reduce_partials", 16.0 * (double)words);
      reduce_partials<<<(u32)((words + 255) / 256), 256, 0, ctx->stream>>>(d_tern, words, m,
                                                                          ctx->logn, ctx->d_primes);
      post_launch(ctx);
    }
    ctx->counts.additions += (u64)pairs * (shards - 1);
  });
}

int lcl_pair_finish(lcl_context* ctx, const uint64_t* d_tern, size_t pairs, size_t width,
                    size_t k, int reduce, uint64_t* d_out) {
  return guarded([&] {
    const u32 m = ctx->full;
    need(m >= 2, LCL_DEPTH_EXHAUSTED, "no prime left to rescale by");
    if (reduce) {
      need(width > 0 && (width & (width - 1)) == 0, LCL_WIDTH_ERROR,
           "reduction width must be a power of two");
      need(width <= ctx->n / 2, LCL_WIDTH_ERROR, "reduction width exceeds the slot count");
    }
    if (!pairs) return;
    u64* ctA = ctx->ws_ctA.get((u64)pairs * 2 * m * ctx->N());
    relinearize_batch(ctx, d_tern, (u32)pairs, m, ctA);
    rescale_batch(ctx, ctA, (u32)pairs, m, d_out);
    if (reduce) slot_reduce_batch(ctx, d_out, (u32)pairs, m - 1, width, k, d_out);
  });
}

int lcl_masked_aggregate_chunks(lcl_context* ctx, const uint64_t* d_clients,
                                const uint64_t* d_sel, size_t n, size_t chunks, double w_scale,
                                double sel_scale, size_t l, int average, size_t chunk_begin,
                                size_t chunk_end, uint64_t* d_out, double* out_scale) {
  return guarded([&] {
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    need(chunk_begin <= chunk_end && chunk_end <= chunks, LCL_SHAPE_ERROR,
         "chunk range outside the weights");
    if (chunk_end > chunk_begin)
      masked_aggregate(ctx, d_clients, d_sel, (u32)n, (u32)chunks, l, average != 0, d_out,
                       (u32)chunk_begin, (u32)chunk_end);
    if (out_scale) {
      double s = (w_scale * sel_scale) / (double)ctx->primes[ctx->full - 1];
      if (average) s = (s * ctx->scale) / (double)ctx->primes[ctx->full - 2];
      *out_scale = s;
    }
  });
}

int lcl_masked_aggregate(lcl_context* ctx, const uint64_t* d_clients, const uint64_t* d_sel,
                         size_t n, size_t chunks, double w_scale, double sel_scale, size_t l,
                         int average, uint64_t* d_out, double* out_scale) {
  return guarded([&] {
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    masked_aggregate(ctx, d_clients, d_sel, (u32)n, (u32)chunks, l, average != 0, d_out);
    if (out_scale) {
      double s = (w_scale * sel_scale) / (double)ctx->primes[ctx->full - 1];
      if (average) s = (s * ctx->scale) / (double)ctx->primes[ctx->full - 2];
      *out_scale = s;
    }
  });
}

int lcl_server_round(lcl_context* ctx, const uint64_t* d_clients, const uint64_t* d_sel,
                     size_t n, size_t chunks, size_t width, size_t k, size_t l, int average,
                     uint64_t* d_dist, uint64_t* d_agg) {
  return guarded([&] {
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    // masked_aggregate on its own lane, forked before the distance matrix:
    // its HBM-bound tensor and short key-switch chain overlap the FP64-bound
    // pair accumulation and the slot_reduce ladder on the context stream
    // (lanes 0 and 1 stay free for slot_reduce)
    if (ctx->prof_on) {
      distance_matrix(ctx, d_clients, (u32)n, (u32)chunks, width, k, true, true, d_dist);
      masked_aggregate(ctx, d_clients, d_sel, (u32)n, (u32)chunks, l, average != 0, d_agg);
      return;
    }
    ensure_lanes(ctx, 3);
    auto& ln = ctx->lanes[2];
    cuda_check(cudaEventRecord(ctx->fork_ev, ctx->stream), "fork");
    cuda_check(cudaStreamWaitEvent(ln.stream, ctx->fork_ev, 0), "lane wait");
    on_lane(ctx, 2, [&] {
      masked_aggregate(ctx, d_clients, d_sel, (u32)n, (u32)chunks, l, average != 0, d_agg);
    });
    cuda_check(cudaEventRecord(ln.done, ln.stream), "lane done");
    distance_matrix(ctx, d_clients, (u32)n, (u32)chunks, width, k, true, true, d_dist);
    cuda_check(cudaStreamWaitEvent(ctx->stream, ln.done, 0), "join");
  });
}

}  // extern "C"

namespace {

// ------------------------------------------------------------ LCLT ingest
// CkksContext::deserialize's header checks (ckks.cpp:640-660), on the host
// (13 bytes per blob); the payload's residue checks run on the device
// (lclt_unpack). Returns the limb count; *scale = 2^scale_bits.
u32 lclt_header(const lcl_context* c, const uint8_t* b, size_t size, double* scale) {
  static const uint8_t magic[4] = {'L', 'C', 'L', 'T'};
  if (size < 13 || std::memcmp(b, magic, 4) != 0) fail(LCL_DATA_ERROR, "not a ciphertext blob");
  if ((u32)(b[4] | (b[5] << 8)) != 1) fail(LCL_DATA_ERROR, "unsupported ciphertext format version");
  const u64 n = (u64)b[6] | ((u64)b[7] << 8) | ((u64)b[8] << 16) | ((u64)b[9] << 24);
  if (n != c->N()) fail(LCL_DATA_ERROR, "ciphertext ring degree does not match the context");
  const u32 level = b[10], scale_bits = b[11], count = b[12];
  if (level > c->full - 1 || count != level + 1)
    fail(LCL_DATA_ERROR, "ciphertext level inconsistent with the modulus chain");
  if (size != 13 + 2ull * count * n * 8) fail(LCL_DATA_ERROR, "ciphertext blob length mismatch");
  if (scale) *scale = std::pow(2.0, (double)scale_bits);
  return count;
}

// Where a host round's inputs come from: limb-major words (the reference's
// PolyRns rows), or LCLT blobs as the server receives them (run_round step
// 3 deserializes every chunk, protocol.cpp:419-429). Blob (i, c) of the
// clients sits at blobs + (i * C + c) * stride, selector i at sel_blobs + i *
// stride. Blob bytes are copied verbatim into a device staging buffer and
// unpacked + range-checked by lclt_unpack on the copy stream, so
// deserialization rides the same overlapped H2D pipeline as plain words.
struct Ingest {
  const u64* words = nullptr;
  const u64* sel_words = nullptr;
  const uint8_t* blobs = nullptr;
  const uint8_t* sel_blobs = nullptr;
  u64 stride = 0;
  u8* stage = nullptr;
  u8* sel_stage = nullptr;
  u32* err = nullptr;  // device: first bad blob (UINT_MAX: none); selectors use err + 1

  void unpack(lcl_context* c, const u8* st, u32 cols, u32 r0, u32 r1, u32 c0, u32 c1, u64* out,
              u32* e, cudaStream_t s) const {
    const u32 m = c->full;
    const u64 W = 2ull * m * c->N();
    const dim3 grid((u32)((W + 255) / 256), (r1 - r0) * (c1 - c0));
    if (!grid.y) return;
    lclt_unpack<<<grid, 256, 0, s>>>(st, stride, cols, r0, c0, c1 - c0, m, c->logn, out, e,
                                     c->d_primes);
    count_launch(c);
    cuda_check(cudaGetLastError(), "lclt_unpack");
  }
  // clients [i0, i1), every chunk
  // clients [i0, i1), every chunk; with an unpack stream u (LCLT blobs), the
  // copy stream records `copied` and moves on while u unpacks the group
  void rows(lcl_context* c, u64* dc, u32 i0, u32 i1, u32 C, cudaStream_t s,
            cudaStream_t u = nullptr, cudaEvent_t copied = nullptr) const {
    const u64 ctw = 2ull * c->full * c->N();
    if (words) {
      cuda_check(cudaMemcpyAsync(dc + (u64)i0 * C * ctw, words + (u64)i0 * C * ctw,
                                 (u64)(i1 - i0) * C * ctw * 8, cudaMemcpyHostToDevice, s), "h2d");
      return;
    }
    cuda_check(cudaMemcpyAsync(stage + (u64)i0 * C * stride, blobs + (u64)i0 * C * stride,
                               (u64)(i1 - i0) * C * stride, cudaMemcpyHostToDevice, s), "h2d blobs");
    if (u) {
      cuda_check(cudaEventRecord(copied, s), "event");
      cuda_check(cudaStreamWaitEvent(u, copied, 0), "wait");
    }
    unpack(c, stage, C, i0, i1, 0, C, dc, err, u ? u : s);
  }
  // chunks [c0, c1) of clients [i0, i1) (one pitched copy), unpacked on u
  // when given (the copy stream records `copied` and moves on)
  void part(lcl_context* c, u64* dc, u32 i0, u32 i1, u32 C, u32 c0, u32 c1, cudaStream_t s,
            cudaStream_t u = nullptr, cudaEvent_t copied = nullptr) const {
    const u64 ctw = 2ull * c->full * c->N();
    if (words) {
      cuda_check(cudaMemcpy2DAsync(dc + ((u64)i0 * C + c0) * ctw, (u64)C * ctw * 8,
                                   words + ((u64)i0 * C + c0) * ctw, (u64)C * ctw * 8,
                                   (u64)(c1 - c0) * ctw * 8, i1 - i0, cudaMemcpyHostToDevice, s),
                 "h2d part");
      return;
    }
    cuda_check(cudaMemcpy2DAsync(stage + ((u64)i0 * C + c0) * stride, (u64)C * stride,
                                 blobs + ((u64)i0 * C + c0) * stride, (u64)C * stride,
                                 (u64)(c1 - c0) * stride, i1 - i0, cudaMemcpyHostToDevice, s),
               "h2d blob part");
    if (u) {
      cuda_check(cudaEventRecord(copied, s), "event");
      cuda_check(cudaStreamWaitEvent(u, copied, 0), "wait");
    }
    unpack(c, stage, C, i0, i1, c0, c1, dc, err, u ? u : s);
  }
  // chunks [c0, c1) of all n clients
  void slice(lcl_context* c, u64* dc, u32 n, u32 C, u32 c0, u32 c1, cudaStream_t s) const {
    const u64 ctw = 2ull * c->full * c->N();
    if (words) {
      cuda_check(cudaMemcpy2DAsync(dc + (u64)c0 * ctw, (u64)C * ctw * 8, words + (u64)c0 * ctw,
                                   (u64)C * ctw * 8, (u64)(c1 - c0) * ctw * 8, n,
                                   cudaMemcpyHostToDevice, s), "h2d slice");
      return;
    }
    cuda_check(cudaMemcpy2DAsync(stage + (u64)c0 * stride, (u64)C * stride, blobs + (u64)c0 * stride,
                                 (u64)C * stride, (u64)(c1 - c0) * stride, n,
                                 cudaMemcpyHostToDevice, s), "h2d blob slice");
    unpack(c, stage, C, 0, n, c0, c1, dc, err, s);
  }
  void sel(lcl_context* c, u64* ds, u32 n, cudaStream_t s) const {
    const u64 ctw = 2ull * c->full * c->N();
    if (sel_words) {
      cuda_check(cudaMemcpyAsync(ds, sel_words, (u64)n * ctw * 8, cudaMemcpyHostToDevice, s), "h2d");
      return;
    }
    cuda_check(cudaMemcpyAsync(sel_stage, sel_blobs, (u64)n * stride, cudaMemcpyHostToDevice, s),
               "h2d sel blobs");
    unpack(c, sel_stage, 1, 0, n, 0, 1, ds, err + 1, s);
  }
};

// Client-group form of the overlapped host round: the clients arrive in G
// groups; when group g has landed, lane g runs the whole chain of the pairs
// it completes (i < j, j in group g: contiguous in j-major order --
// accumulation, relinearize, rescale, slot_reduce, D2H) while later groups
// are still in flight. The aggregate ternaries accumulate group by group (the
// tensor is a sum over clients) and are finished on the last lane. Group
// boundaries k_g ~ n sqrt(g / G) give the lanes similar pair counts. Same
// kernels and op counters as the serial round.
void host_round_groups(lcl_context* ctx, const Ingest& in, u32 n, u32 C,
                       size_t width, size_t k, size_t l, bool average, u64* h_dist, u64* h_agg,
                       u64* dc, u64* ds, u64* dd, u64* da, u32 G) {
  const u32 m = ctx->full;
  const u64 N = ctx->N();
  const u64 dstride = 2ull * (m - 1) * N;
  const u64 astride = 2ull * (average ? m - 2 : m - 1) * N;
  // The last T clients arrive as single-client groups (LCL_TAIL_SINGLES; by
  // default n / 4 when one client's bytes take >= ~10 ms of PCIe): a single
  // client's chain (its pairs' accumulation and key-switch ladder) then
  // fits inside the next client's copy, so only the last client's chain is
  // left after the last byte. The head [0, n - T) is cut by the sqrt rule.
  const int tail_env = [] {
    const char* e = std::getenv("LCL_TAIL_SINGLES");
    return e ? atoi(e) : -1;
  }();
  const u64 client_bytes = (u64)C * 2 * m * N * 8;
  u32 T = tail_env >= 0 ? (u32)tail_env : (client_bytes >= (512ull << 20) ? n / 4 : 0);
  T = std::min(T, n - 2);
  const u32 head = n - T;
  std::vector<u32> bound{0};
  for (u32 g = 1; g < G; ++g) {
    const u32 kb = (u32)std::lround(head * std::sqrt((double)g / G));
    if (kb > bound.back() + 1 && kb < head) bound.push_back(kb);
  }
  bound.push_back(head);
  for (u32 j = head + 1; j <= n; ++j) bound.push_back(j);
  G = (u32)bound.size() - 1;
  ensure_lanes(ctx, G);
  // With single-client tail groups, the last two lanes (the chains that
  // finish last) run on highest-priority streams, ahead of the other lanes'
  // work and of the last group's slice accumulations (lowest priority), and
  // the aggregate slices too (LCL_LANE_PRIO = 0 / 1 forces it off / on;
  // cfg3 e2e 541.4 -> 539.9 ms; at cfg2, with no tail singles, it costs
  // 12.8 -> 13.6 ms, so it follows T by default)
  const int prio_env = [] {
    const char* e = std::getenv("LCL_LANE_PRIO");
    return e ? atoi(e) : -1;
  }();
  const bool prio = prio_env >= 0 ? prio_env == 1 : T > 0;
  if (!ctx->crit) {
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    cuda_check(cudaStreamCreateWithPriority(&ctx->crit, cudaStreamNonBlocking, hi), "stream");
    cuda_check(cudaStreamCreateWithPriority(&ctx->crit2, cudaStreamNonBlocking, hi), "stream");
    cuda_check(cudaStreamCreateWithPriority(&ctx->lo, cudaStreamNonBlocking, lo), "stream");
    cuda_check(cudaStreamCreateWithPriority(&ctx->crit3, cudaStreamNonBlocking, hi), "stream");
  }
  struct LaneSwap {  // swapped back on every exit path
    lcl_context* c;
    u32 g;
    bool on;
    ~LaneSwap() {
      if (!on) return;
      std::swap(c->lanes[g].stream, c->crit);
      if (g) std::swap(c->lanes[g - 1].stream, c->crit2);
    }
  } lane_swap{ctx, G - 1, prio};
  if (prio) {
    std::swap(ctx->lanes[G - 1].stream, ctx->crit);
    if (G >= 2) std::swap(ctx->lanes[G - 2].stream, ctx->crit2);
  }
  while (ctx->io_ev.size() < 1 + 3 * (size_t)G) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ctx->io_ev.push_back(e);
  }
  // events: 0 start; 1+g group g landed; 1+G+g its aggregate part; 1+2G+g lane done
  cudaEvent_t* ev = ctx->io_ev.data();
  const u64* d_pt = average ? agg_plaintext(ctx, l) : nullptr;
  cuda_check(cudaEventRecord(ev[0], ctx->stream), "event");
  cuda_check(cudaStreamWaitEvent(ctx->h2d, ev[0], 0), "wait");
  cuda_check(cudaStreamWaitEvent(ctx->d2h, ev[0], 0), "wait");
  cuda_check(cudaStreamWaitEvent(ctx->d2h_agg, ev[0], 0), "wait");
  for (u32 g = 0; g < G; ++g) cuda_check(cudaStreamWaitEvent(ctx->lanes[g].stream, ev[0], 0), "wait");
  in.sel(ctx, ds, n, ctx->h2d);
  // LCLT groups are unpacked on their own stream so the next group's copy
  // starts as soon as this one's bytes are in (the unpack kernels would
  // otherwise sit between the copies on the copy stream)
  cudaStream_t up = nullptr;
  if (in.blobs) {
    if (!ctx->unpk) {  // highest priority: every later step waits for the unpacked words
      int lo = 0, hi = 0;
      cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
      cuda_check(cudaStreamCreateWithPriority(&ctx->unpk, cudaStreamNonBlocking, hi), "stream");
    }
    while (ctx->unpk_ev.size() < G + 1) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      ctx->unpk_ev.push_back(e);
    }
    up = ctx->unpk;
    // the selectors (unpacked on the copy stream) come first
    cuda_check(cudaEventRecord(ctx->unpk_ev[G], ctx->h2d), "event");
    cuda_check(cudaStreamWaitEvent(up, ctx->unpk_ev[G], 0), "wait");
  }
  // LCL_TRACE_ROUND=1: print when the last byte landed, the last group was
  // unpacked, the lanes finished and the last D2H completed (ms from start)
  static const bool trace = std::getenv("LCL_TRACE_ROUND") != nullptr;
  cudaEvent_t tr[6] = {};
  std::vector<cudaEvent_t> trl;  // per lane: pair accumulation done, chain done
  if (trace) {
    for (auto& e : tr) cuda_check(cudaEventCreate(&e), "trace event");
    trl.resize(2 * G);
    for (auto& e : trl) cuda_check(cudaEventCreate(&e), "trace event");
    cuda_check(cudaEventRecord(tr[0], ctx->stream), "event");
  }
  // The last group can arrive in S chunk slices (LCL_LAST_SLICES, default
  // 8): the aggregate is a sum over every client, so only the last group's
  // bytes hold it back; per slice, the aggregate chunks are finished and
  // copied out while the next slice lands, instead of all 342 chunks'
  // aggregate (1.07 GB D2H at cfg3) after the last byte. LCL_LAST_PAIRS=1
  // also accumulates the last group's pairs slice by slice.
  const int last_slices_env = [] {
    const char* e = std::getenv("LCL_LAST_SLICES");
    return e ? atoi(e) : 8;
  }();
  const bool last_pairs = [] {
    const char* e = std::getenv("LCL_LAST_PAIRS");
    return e && e[0] == '1';
  }();
  const u32 S = G >= 2 && last_slices_env > 1 ? std::min<u32>((u32)last_slices_env, C) : 1;
  while (ctx->io_ev.size() < 1 + 3 * (size_t)G + 2 * S + 4) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ctx->io_ev.push_back(e);
  }
  ev = ctx->io_ev.data();
  cudaEvent_t* sev = ev + 1 + 3 * G;  // slice s landed (and unpacked)
  cudaEvent_t* aev = sev + S;         // slice s's aggregate chunks finished
  cudaEvent_t lfork = aev[S], lacc = aev[S + 1];  // last lane -> slice stream -> last lane
  cudaEvent_t afork = aev[S + 2], ajoin = aev[S + 3];  // lane 0 -> aggregate slices -> lane 0
  // Runs f with the context's stream replaced by s, ordered after and
  // joined back into the current stream (lane workspaces stay the lane's).
  auto on_stream = [&](cudaStream_t st, cudaEvent_t fork, cudaEvent_t join, auto&& f) {
    cudaStream_t own = ctx->stream;
    cuda_check(cudaEventRecord(fork, own), "event");
    cuda_check(cudaStreamWaitEvent(st, fork, 0), "wait");
    ctx->stream = st;
    try {
      f();
    } catch (...) {
      ctx->stream = own;
      throw;
    }
    ctx->stream = own;
    cuda_check(cudaEventRecord(join, st), "event");
    cuda_check(cudaStreamWaitEvent(own, join, 0), "wait");
  };
  if (in.blobs) {
    while (ctx->unpk_ev.size() < G + 1 + S) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      ctx->unpk_ev.push_back(e);
    }
  }
  auto slice_lo = [&](u32 s) { return (u32)((u64)C * s / S); };
  for (u32 g = 0; g < G; ++g) {
    if (g + 1 == G && S > 1) {
      for (u32 s = 0; s < S; ++s) {
        in.part(ctx, dc, bound[g], bound[g + 1], C, slice_lo(s), slice_lo(s + 1), ctx->h2d, up,
                up ? ctx->unpk_ev[G + 1 + s] : nullptr);
        cuda_check(cudaEventRecord(sev[s], up ? up : ctx->h2d), "event");
      }
    } else {
      in.rows(ctx, dc, bound[g], bound[g + 1], C, ctx->h2d, up, up ? ctx->unpk_ev[g] : nullptr);
    }
    cuda_check(cudaEventRecord(ev[1 + g], up ? up : ctx->h2d), "event");
  }
  if (trace) {
    cuda_check(cudaEventRecord(tr[1], ctx->h2d), "event");
    cuda_check(cudaEventRecord(tr[2], up ? up : ctx->h2d), "event");
  }
  u64* atern = ctx->ws_atern.get((u64)C * 3 * m * N);
  const u32 P = n * (n - 1) / 2;
  u64* tern = ctx->ws_dtern.get((u64)P * 3 * m * N);  // j-major, disjoint per group
  u32 first = 0;  // j-major index of the group's first pair
  for (u32 g = 0; g < G; ++g) {
    const PairSet ps = completed_by(bound[g], bound[g + 1]);
    const u32 B = pair_count(n, ps);
    u64* o = dd + (u64)first * dstride;
    u64* t = tern + (u64)first * 3 * m * N;
    if (g + 1 == G && S > 1) {
      // the last group's aggregate slices on lane 0 (its own chain is long
      // done): tensor of the group's clients onto the earlier groups' sums,
      // relinearize + rescale, D2H on the aggregate's copy stream
      on_lane(ctx, 0, [&] { on_stream(prio ? ctx->crit3 : ctx->stream, afork, ajoin, [&] {
        cuda_check(cudaStreamWaitEvent(ctx->stream, ev[G + g], 0), "wait");
        for (u32 s = 0; s < S; ++s) {
          const u32 c0 = slice_lo(s), c1 = slice_lo(s + 1);
          cuda_check(cudaStreamWaitEvent(ctx->stream, sev[s], 0), "wait");
          agg_tensor(ctx, dc, ds, n, C, c0, c1 - c0, bound[g], bound[g + 1],
                     atern + (u64)c0 * 3 * m * N, true);
          for (u32 b0 = c0; b0 < c1; b0 += sub_batch(ctx, m)) {
            const u32 Bc = std::min(c1, b0 + sub_batch(ctx, m)) - b0;
            agg_finish(ctx, atern + (u64)b0 * 3 * m * N, Bc, average, d_pt, da + (u64)b0 * astride);
          }
          cuda_check(cudaEventRecord(aev[s], ctx->stream), "event");
          cuda_check(cudaStreamWaitEvent(ctx->d2h_agg, aev[s], 0), "wait");
          cuda_check(cudaMemcpyAsync(h_agg + (u64)c0 * astride, da + (u64)c0 * astride,
                                     (u64)(c1 - c0) * astride * 8, cudaMemcpyDeviceToHost,
                                     ctx->d2h_agg), "d2h agg slice");
        }
        cuda_check(cudaEventRecord(ev[1 + G + g], ctx->stream), "event");
      }); });
      on_lane(ctx, g, [&] {
        if (B) {
          if (last_pairs) {
            // slice accumulations on the lowest-priority stream (they have
            // slack until the last byte); the chain continues on the lane
            on_stream(prio ? ctx->lo : ctx->stream, lfork, lacc, [&] {
              for (u32 s = 0; s < S; ++s) {
                cuda_check(cudaStreamWaitEvent(ctx->stream, sev[s], 0), "wait");
                pair_accumulate_launch(ctx, dc, n, C, slice_lo(s), slice_lo(s + 1), ps, t, s > 0);
              }
            });
          } else {
            cuda_check(cudaStreamWaitEvent(ctx->stream, ev[1 + g], 0), "wait");
            pair_accumulate_launch(ctx, dc, n, C, 0, C, ps, t, false);
          }
          if (trace) cuda_check(cudaEventRecord(trl[2 * g], ctx->stream), "event");
          u64* ctA = ctx->ws_ctA.get((u64)B * 2 * m * N);
          relinearize_batch(ctx, t, B, m, ctA);
          rescale_batch(ctx, ctA, B, m, o);
          slot_reduce_batch(ctx, o, B, m - 1, width, k, o);
        }
        if (trace) cuda_check(cudaEventRecord(trl[2 * g + 1], ctx->stream), "event");
        cuda_check(cudaEventRecord(ev[1 + 2 * G + g], ctx->stream), "event");
      });
    } else
    on_lane(ctx, g, [&] {
      cuda_check(cudaStreamWaitEvent(ctx->stream, ev[1 + g], 0), "wait");
      if (g > 0) cuda_check(cudaStreamWaitEvent(ctx->stream, ev[G + g], 0), "wait");
      for (u32 c0 = 0; c0 < C; c0 += 32768)
        agg_tensor(ctx, dc, ds, n, C, c0, std::min(C, c0 + 32768) - c0, bound[g], bound[g + 1],
                   atern + (u64)c0 * 3 * m * N, g > 0);
      if (g + 1 < G) {
        cuda_check(cudaEventRecord(ev[1 + G + g], ctx->stream), "event");
      } else {
        // (finishing the aggregate on lane 0 beside this lane's pair chain
        // measured slower: cfg3 e2e 577.6 vs 566.2 ms at 8 groups)
        for (u32 c0 = 0; c0 < C; c0 += sub_batch(ctx, m)) {
          const u32 Bc = std::min(C, c0 + sub_batch(ctx, m)) - c0;
          agg_finish(ctx, atern + (u64)c0 * 3 * m * N, Bc, average, d_pt, da + (u64)c0 * astride);
        }
        cuda_check(cudaEventRecord(ev[1 + G + g], ctx->stream), "event");
        // on its own stream: the D2H stream's earlier pair copies wait for
        // the other lanes' chains, which would hold the aggregate back
        cuda_check(cudaStreamWaitEvent(ctx->d2h_agg, ev[1 + G + g], 0), "wait");
        cuda_check(cudaMemcpyAsync(h_agg, da, (u64)C * astride * 8, cudaMemcpyDeviceToHost,
                                   ctx->d2h_agg), "d2h agg");
      }
      if (B) {
        pair_accumulate_launch(ctx, dc, n, C, 0, C, ps, t, false);
        if (trace) cuda_check(cudaEventRecord(trl[2 * g], ctx->stream), "event");
        u64* ctA = ctx->ws_ctA.get((u64)B * 2 * m * N);
        relinearize_batch(ctx, t, B, m, ctA);
        rescale_batch(ctx, ctA, B, m, o);
        slot_reduce_batch(ctx, o, B, m - 1, width, k, o);
      }
      if (trace) cuda_check(cudaEventRecord(trl[2 * g + 1], ctx->stream), "event");
      cuda_check(cudaEventRecord(ev[1 + 2 * G + g], ctx->stream), "event");
    });
    cuda_check(cudaStreamWaitEvent(ctx->d2h, ev[1 + 2 * G + g], 0), "wait");
    // j-major group order -> the matrix's row-major (i < j) slots
    u32 q = 0;
    for (u32 j = bound[g]; j < bound[g + 1]; ++j)
      for (u32 i = 0; i < j; ++i, ++q) {
        const u64 p = (u64)i * (2ull * n - i - 1) / 2 + (j - i - 1);
        cuda_check(cudaMemcpyAsync(h_dist + p * dstride, o + (u64)q * dstride, dstride * 8,
                                   cudaMemcpyDeviceToHost, ctx->d2h), "d2h pair");
      }
    first += B;
  }
  ctx->counts.multiplications += (u64)P * C + (u64)n * C;
  ctx->counts.additions += (u64)P * (2ull * C - 1) + (u64)(n - 1) * C;
  for (u32 g = 0; g < G; ++g)
    cuda_check(cudaStreamWaitEvent(ctx->stream, ev[1 + 2 * G + g], 0), "join");
  // the aggregate's last part (on lane 0 when the last group is sliced)
  cuda_check(cudaStreamWaitEvent(ctx->stream, ev[2 * G], 0), "join aggregate");
  if (trace) {
    cuda_check(cudaEventRecord(tr[3], ctx->stream), "event");
    cuda_check(cudaEventRecord(tr[4], ctx->d2h), "event");
    cuda_check(cudaEventRecord(tr[5], ctx->d2h_agg), "event");
  }
  cuda_check(cudaStreamSynchronize(ctx->d2h_agg), "round sync");
  cuda_check(cudaStreamSynchronize(ctx->d2h), "round sync");
  cuda_check(cudaStreamSynchronize(ctx->stream), "round sync");
  if (trace) {
    float t[5];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], tr[0], tr[i + 1]);
    std::fprintf(stderr,
                 "host round (G=%u): last byte %.2f ms, last unpack %.2f, lanes done %.2f, pair d2h done %.2f, "
                 "aggregate d2h done %.2f\n",
                 G, t[0], t[1], t[2], t[3], t[4]);
    for (u32 g = 0; g < G; ++g) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, tr[0], trl[2 * g]);
      cudaEventElapsedTime(&b, tr[0], trl[2 * g + 1]);
      std::fprintf(stderr, "  lane %u (clients %u..%u, %u pairs): accumulated %.2f ms, chain done %.2f\n", g,
                   bound[g], bound[g + 1] - 1, pair_count(n, completed_by(bound[g], bound[g + 1])), a, b);
    }
    for (auto& e : trl) cudaEventDestroy(e);
    for (auto& e : tr) cudaEventDestroy(e);
  }
}

// lcl_server_round_host / lcl_server_round_lclt: H2D (words or LCLT blobs),
// the round, D2H; see the header.
void server_round_host(lcl_context* ctx, const Ingest& in, size_t n, size_t chunks, size_t width,
                       size_t k, size_t l, int average, uint64_t* h_dist, uint64_t* h_agg) {
  {
    const u32 m = ctx->full;
    const u64 N = ctx->N();
    const u64 ctw = 2ull * m * N;  // words per ciphertext
    const u64 cw = (u64)n * chunks * ctw, sw = (u64)n * ctw;
    const u32 P = (u32)(n * (n - 1) / 2);
    const u64 dstride = 2ull * (m - 1) * N;
    const u64 astride = 2ull * (average ? m - 2 : m - 1) * N;
    const u64 dw = (u64)P * dstride, aw = (u64)chunks * astride;
    u64* dc = ctx->ws_io_in.get(cw);
    u64* ds = ctx->ws_io_sel.get(sw);
    u64* dd = ctx->ws_io_dist.get(dw);
    u64* da = ctx->ws_io_agg.get(aw);
    const bool overlap = n >= 2 && n <= 65535 && m >= 2 && chunks >= 2 && P <= sub_batch(ctx, m);
    (void)sw;
    if (!overlap) {
      in.rows(ctx, dc, 0, (u32)n, (u32)chunks, ctx->stream);
      in.sel(ctx, ds, (u32)n, ctx->stream);
      distance_matrix(ctx, dc, (u32)n, (u32)chunks, width, k, true, true, dd);
      masked_aggregate(ctx, dc, ds, (u32)n, (u32)chunks, l, average != 0, da);
      cuda_check(cudaMemcpyAsync(h_dist, dd, dw * 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
      cuda_check(cudaMemcpyAsync(h_agg, da, aw * 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
      cuda_check(cudaStreamSynchronize(ctx->stream), "round sync");
      return;
    }
    // Overlapped round (LCLT ingest): the clients arrive in chunk
    // slices on an H2D stream; slice s is accumulated into every pair's
    // ternary and aggregated (tensor, relinearize, rescale of its chunks)
    // while slice s + 1 is in flight, and its aggregate chunks leave on a D2H
    // stream. The pair chains (relinearize, rescale, slot_reduce) follow the
    // last slice. Same kernels and op counters as distance_matrix +
    // masked_aggregate, so the words are identical. (A client-major order --
    // start the chains of the pairs a client group completes -- was measured
    // too: 17.1 ms at cfg2, where a 10-pair chain costs nearly as much as the
    // 45-pair one, and 575 vs 584 ms at cfg3, where the H2D dominates.)
    if (width == 0 || (width & (width - 1))) fail(LCL_WIDTH_ERROR, "reduction width must be a power of two");
    if (width > ctx->n / 2) fail(LCL_WIDTH_ERROR, "reduction width exceeds the slot count");
    if (average && m < 3) fail(LCL_DEPTH_EXHAUSTED, "no prime left to rescale by");
    if (!ctx->d_relin) fail(LCL_KEY_ERROR, "no relinearization key uploaded");
    ensure_pairs(ctx, (u32)n);
    if (!ctx->h2d) cuda_check(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking), "stream");
    if (!ctx->d2h) cuda_check(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking), "stream");
    if (!ctx->d2h_agg) cuda_check(cudaStreamCreateWithFlags(&ctx->d2h_agg, cudaStreamNonBlocking), "stream");
    // 0: chunk slices, 1: 2 client groups, G >= 2: G groups (read per call).
    // Default 8 groups: the smaller the last group, the shorter the chain
    // left after the last byte lands -- e2e cfg3 592.5 (2 groups), 574.4 (4),
    // 568.9 (6), 566.2 (8), 567.8 ms (10); cfg2 13.17 / 14.06 / 12.81 / 12.66
    // / 13.55 ms. Round 2, with 32 hardware queues (CUDA_DEVICE_MAX_CONNECTIONS,
    // set by the package: with 8, lanes alias onto the copy streams' queues),
    // the last group in 8 chunk slices for the aggregate (549.4 ms), the last
    // n / 4 clients as single-client groups and the last lanes at high
    // priority: cfg3 e2e 556.9 -> ~540 ms; cfg2 unchanged (no tail singles).
    // Rejected: the last client's pairs accumulated per slice (LCL_LAST_PAIRS=1,
    // 541-551 ms: the slices starve the second-to-last chain), 2 or 4 slots
    // per thread in the pair kernel for small pair sets (683 / 562 ms).
    const char* mode_env = std::getenv("LCL_HOST_ROUND");
    const int mode = mode_env ? atoi(mode_env) : 8;
    if (mode >= 1 && ctx->pair_f64 && n >= 4 && !ctx->prof_on) {
      host_round_groups(ctx, in, (u32)n, (u32)chunks, width, k, l, average != 0,
                        h_dist, h_agg, dc, ds, dd, da, mode == 1 ? 2u : (u32)mode);
      return;
    }
    const u32 C = (u32)chunks;
    const u32 slices = std::min<u32>(C, 16);
    const u32 per = (C + slices - 1) / slices;
    while (ctx->io_ev.size() < 2 * (size_t)slices + 2) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      ctx->io_ev.push_back(e);
    }
    cudaEvent_t* ev = ctx->io_ev.data();
    cudaEvent_t start = ev[2 * slices], dist_done = ev[2 * slices + 1];
    // copies start after whatever the compute stream already holds
    cuda_check(cudaEventRecord(start, ctx->stream), "event");
    cuda_check(cudaStreamWaitEvent(ctx->h2d, start, 0), "wait");
    cuda_check(cudaStreamWaitEvent(ctx->d2h, start, 0), "wait");
    in.sel(ctx, ds, (u32)n, ctx->h2d);
    u64* tern = ctx->ws_dtern.get((u64)P * 3 * m * N);
    u32 s = 0;
    for (u32 c0 = 0; c0 < C; c0 += per, ++s) {
      const u32 c1 = std::min(C, c0 + per);
      // clients' chunks [c0, c1): n rows of (c1 - c0) ciphertexts, pitch C
      in.slice(ctx, dc, (u32)n, C, c0, c1, ctx->h2d);
      cuda_check(cudaEventRecord(ev[2 * s], ctx->h2d), "event");
      cuda_check(cudaStreamWaitEvent(ctx->stream, ev[2 * s], 0), "wait");
      pair_accumulate_launch(ctx, dc, (u32)n, C, c0, c1, row_range(0, P), tern, c0 > 0);
      masked_aggregate(ctx, dc, ds, (u32)n, C, l, average != 0, da + (u64)c0 * astride, c0, c1);
      cuda_check(cudaEventRecord(ev[2 * s + 1], ctx->stream), "event");
      cuda_check(cudaStreamWaitEvent(ctx->d2h, ev[2 * s + 1], 0), "wait");
      cuda_check(cudaMemcpyAsync(h_agg + (u64)c0 * astride, da + (u64)c0 * astride,
                                 (u64)(c1 - c0) * astride * 8, cudaMemcpyDeviceToHost, ctx->d2h),
                 "d2h slice");
    }
    ctx->counts.multiplications += (u64)P * C;
    ctx->counts.additions += (u64)P * (2ull * C - 1);
    u64* ctA = ctx->ws_ctA.get((u64)P * 2 * m * N);
    relinearize_batch(ctx, tern, P, m, ctA);
    rescale_batch(ctx, ctA, P, m, dd);
    slot_reduce_batch(ctx, dd, P, m - 1, width, k, dd);
    cuda_check(cudaEventRecord(dist_done, ctx->stream), "event");
    cuda_check(cudaStreamWaitEvent(ctx->d2h, dist_done, 0), "wait");
    cuda_check(cudaMemcpyAsync(h_dist, dd, dw * 8, cudaMemcpyDeviceToHost, ctx->d2h), "d2h");
    cuda_check(cudaStreamSynchronize(ctx->d2h), "round sync");
    cuda_check(cudaStreamSynchronize(ctx->stream), "round sync");
  }
}

// Validates the headers of a batch of LCLT blobs on the host: all at the
// same limb count (returned) and scale (*scale).
u32 lclt_batch_headers(const lcl_context* c, const uint8_t* blobs, size_t blob_bytes,
                       size_t stride, size_t count, double* scale) {
  need(stride >= blob_bytes, LCL_SHAPE_ERROR, "blob stride shorter than a blob");
  u32 m = 0;
  for (size_t i = 0; i < count; ++i) {
    double sc = 0;
    const u32 mi = lclt_header(c, blobs + i * stride, blob_bytes, &sc);
    if (i == 0) {
      m = mi;
      *scale = sc;
    }
    need(mi == m, LCL_SHAPE_ERROR, "blobs of one batch differ in level");
    need(sc == *scale, LCL_ALIGNMENT_ERROR, "operand scales diverge");
  }
  return m;
}

// Reads back the unpack kernels' first-bad-blob words (synchronises).
void lclt_check(lcl_context* c, const u32* d_err, int words) {
  u32 h[2] = {0xFFFFFFFFu, 0xFFFFFFFFu};
  cuda_check(cudaMemcpy(h, d_err, (size_t)words * 4, cudaMemcpyDeviceToHost), "err readback");
  for (int i = 0; i < words; ++i)
    if (h[i] != 0xFFFFFFFFu) fail(LCL_DATA_ERROR, "residue outside its modulus");
}

}  // namespace

extern "C" {

int lcl_server_round_host(lcl_context* ctx, const uint64_t* h_clients, const uint64_t* h_sel,
                          size_t n, size_t chunks, double in_scale, size_t width, size_t k,
                          size_t l, int average, uint64_t* h_dist, uint64_t* h_agg) {
  return guarded([&] {
    Ingest in;
    in.words = h_clients;
    in.sel_words = h_sel;
    server_round_host(ctx, in, n, chunks, width, k, l, average, h_dist, h_agg);
    (void)in_scale;
  });
}

int lcl_server_round_lclt(lcl_context* ctx, const uint8_t* h_client_blobs,
                          const uint8_t* h_sel_blobs, size_t blob_bytes, size_t stride, size_t n,
                          size_t chunks, size_t width, size_t k, size_t l, int average,
                          uint64_t* h_dist, uint64_t* h_agg, double* dist_scale,
                          double* agg_scale) {
  return guarded([&] {
    need(chunks >= 1, LCL_SHAPE_ERROR, "empty weight vector");
    double w_scale = 0, s_scale = 0;
    const u32 m = lclt_batch_headers(ctx, h_client_blobs, blob_bytes, stride, n * chunks, &w_scale);
    const u32 ms = lclt_batch_headers(ctx, h_sel_blobs, blob_bytes, stride, n, &s_scale);
    need(m == ctx->full && ms == ctx->full, LCL_SHAPE_ERROR,
         "client updates and selectors must be fresh (top-level) ciphertexts");
    Ingest in;
    in.blobs = h_client_blobs;
    in.sel_blobs = h_sel_blobs;
    in.stride = stride;
    // staging: the blob bytes verbatim (+16: the funnel shift's last load)
    in.stage = reinterpret_cast<u8*>(ctx->ws_stage.get((n * chunks * stride + 16 + 7) / 8));
    in.sel_stage = reinterpret_cast<u8*>(ctx->ws_stage_sel.get((n * stride + 16 + 7) / 8));
    in.err = reinterpret_cast<u32*>(ctx->ws_err.get(1));
    cuda_check(cudaMemsetAsync(in.err, 0xFF, 8, ctx->stream), "err reset");
    server_round_host(ctx, in, n, chunks, width, k, l, average, h_dist, h_agg);
    lclt_check(ctx, in.err, 2);
    const u32 full = ctx->full;
    if (dist_scale) *dist_scale = (w_scale * w_scale) / (double)ctx->primes[full - 1];
    if (agg_scale) {
      double sc = (w_scale * s_scale) / (double)ctx->primes[full - 1];
      if (average) sc = (sc * ctx->scale) / (double)ctx->primes[full - 2];
      *agg_scale = sc;
    }
  });
}

int lcl_deserialize(lcl_context* ctx, const uint8_t* h_blobs, size_t blob_bytes, size_t stride,
                    size_t count, uint64_t* d_out, double* scale) {
  return guarded([&] {
    if (!count) return;
    double sc = 0;
    lclt_batch_headers(ctx, h_blobs, blob_bytes, stride, count, &sc);
    u8* st = reinterpret_cast<u8*>(ctx->ws_stage.get((count * stride + 16 + 7) / 8));
    u32* err = reinterpret_cast<u32*>(ctx->ws_err.get(1));
    cuda_check(cudaMemsetAsync(err, 0xFF, 8, ctx->stream), "err reset");
    cuda_check(cudaMemcpyAsync(st, h_blobs, count * stride, cudaMemcpyHostToDevice, ctx->stream),
               "h2d blobs");
    const u32 m = h_blobs[12];
    const u64 W = 2ull * m * ctx->N();
    const dim3 grid((u32)((W + 255) / 256), (u32)count);
    lclt_unpack<<<grid, 256, 0, ctx->stream>>>(st, stride, (u32)count, 0, 0, (u32)count, m,
                                               ctx->logn, d_out, err, ctx->d_primes);
    post_launch(ctx);
    cuda_check(cudaStreamSynchronize(ctx->stream), "deserialize sync");
    lclt_check(ctx, err, 1);
    if (scale) *scale = sc;
  });
}

int lcl_serialize(lcl_context* ctx, const uint64_t* d_ct, size_t count, size_t limbs,
                  double scale, uint8_t* h_blobs, size_t stride) {
  return guarded([&] {
    check_count(ctx, limbs);
    const long long sb = std::llround(std::log2(scale));
    need(sb >= 1 && sb <= 255, LCL_PARAMETER_ERROR, "scale exponent does not fit the header");
    const u64 W = 2ull * limbs * ctx->N();
    const u64 bytes = 13 + 8 * W;
    need(stride >= bytes, LCL_SHAPE_ERROR, "blob stride shorter than a blob");
    if (!count) return;
    u8* st = reinterpret_cast<u8*>(ctx->ws_stage.get((count * stride + 7) / 8));
    const dim3 grid((u32)((W + 255) / 256), (u32)count);
    lclt_pack<<<grid, 256, 0, ctx->stream>>>(d_ct, (u32)limbs, ctx->logn, (u32)limbs - 1, (u32)sb,
                                             stride, st);
    post_launch(ctx);
    cuda_check(cudaMemcpyAsync(h_blobs, st, count * stride, cudaMemcpyDeviceToHost, ctx->stream),
               "d2h blobs");
    cuda_check(cudaStreamSynchronize(ctx->stream), "serialize sync");
  });
}

}  // extern "C"
