// lancelot_b200.hpp — C++ mirror of the reference's server API over the C-ABI.
//
// For C++ callers of the reference (lancelot::core, /root/reference/proj/core)
// this header keeps the names, argument meaning and exception types of
//   build_distance_matrix   distance.hpp:123-126
//   masked_aggregate        aggregation.hpp:90-93
//   HoistPlan / slot_reduce_steps / fixed_plan       distance.hpp:67-99
//   errors                  errors.hpp:27-104
// while the work runs on the B200 through include/lancelot_b200.h. Two layers:
//   * reference-signature API (below "drop-in"): host-side Ciphertext /
//     PackedWeights / RelinKey / RotationKeySet / SelectionMask with the
//     reference's member names, and build_distance_matrix / masked_aggregate
//     with the reference's exact parameter lists, so the reference's own call
//     sites (protocol.cpp:430-432, 492-493) compile unchanged against it;
//   * device-resident API (ClientBatch, DeviceBuffer): the same work on
//     ciphertext batches already in HBM (no per-call H2D), used by servers
//     that keep the round resident.
// The layouts are the reference's (limb-major u64, c0 rows then c1 rows).
// Threading: the reference shares one const CkksContext across threads
// (atomic counters, mutex-guarded caches). An lcl_context is NOT thread-safe
// (one stream, shared workspaces); this mirror serialises every call on a
// context with a mutex, so a const CkksContext may be shared the same way.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lancelot_b200.h"

namespace lancelot_b200 {

// ------------------------------------------------------------------ errors
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
#define LCL_ERR(Name) \
  class Name : public Error { \
   public: \
    using Error::Error; \
  };
LCL_ERR(ParameterError)
LCL_ERR(BasisMismatchError)
LCL_ERR(DomainError)
LCL_ERR(AlignmentError)
LCL_ERR(KeyError)
LCL_ERR(DepthExhaustedError)
LCL_ERR(CapacityError)
LCL_ERR(ShapeError)
LCL_ERR(WidthError)
LCL_ERR(InfeasibleError)
LCL_ERR(DataError)
LCL_ERR(UsageError)
LCL_ERR(DeviceError)
#undef LCL_ERR

inline void check(int rc) {
  if (rc == LCL_OK) return;
  const std::string m = lcl_last_error();
  switch (rc) {
    case LCL_PARAMETER_ERROR: throw ParameterError(m);
    case LCL_BASIS_MISMATCH: throw BasisMismatchError(m);
    case LCL_DOMAIN_ERROR: throw DomainError(m);
    case LCL_ALIGNMENT_ERROR: throw AlignmentError(m);
    case LCL_KEY_ERROR: throw KeyError(m);
    case LCL_DEPTH_EXHAUSTED: throw DepthExhaustedError(m);
    case LCL_CAPACITY_ERROR: throw CapacityError(m);
    case LCL_SHAPE_ERROR: throw ShapeError(m);
    case LCL_WIDTH_ERROR: throw WidthError(m);
    case LCL_INFEASIBLE_ERROR: throw InfeasibleError(m);
    case LCL_DATA_ERROR: throw DataError(m);
    case LCL_USAGE_ERROR: throw UsageError(m);
    default: throw DeviceError(m);
  }
}

// ------------------------------------------------------------------ plans
struct HoistPlan {  // distance.hpp:70-78, same fields in the same order
  std::size_t k = 1;
  double t_hoist = 0.0;
  double t_decompose = 0.0;
  double m_cipher = 0.0;
  double m_budget = 0.0;
  std::size_t n = 1;
  double cost = 0.0;
};

enum class HoistMode { off, full, dynamic_lp };

inline std::size_t require_width_levels(std::size_t n) {
  if (n == 0 || (n & (n - 1))) throw WidthError("reduction width must be a power of two");
  std::size_t levels = 0;
  while ((std::size_t{1} << levels) < n) ++levels;
  return levels;
}

// plan_unfold (distance.cpp:144-179): exhaustive minimisation of
// (log2 n - k + 1) t_hoist + (k - 1) t_decompose over k * m_cipher <= budget.
inline HoistPlan plan_unfold(double t_hoist, double t_decompose, double m_cipher,
                             double m_budget, std::size_t n) {
  if (!(t_hoist > 0.0) || !(t_decompose > 0.0) || !(m_cipher > 0.0) || !(m_budget > 0.0))
    throw ParameterError("plan inputs must all be positive");
  const std::size_t levels = require_width_levels(n);
  if (m_cipher > m_budget) throw InfeasibleError("one ciphertext already exceeds the memory budget");
  const double mem_cap = std::floor(m_budget / m_cipher);
  std::size_t k_max = levels + 1;
  if (mem_cap < static_cast<double>(k_max)) k_max = static_cast<std::size_t>(mem_cap);
  HoistPlan plan;
  plan.t_hoist = t_hoist;
  plan.t_decompose = t_decompose;
  plan.m_cipher = m_cipher;
  plan.m_budget = m_budget;
  plan.n = n;
  plan.k = 1;
  plan.cost = static_cast<double>(levels) * t_hoist;
  for (std::size_t k = 2; k <= k_max; ++k) {
    const double cost = static_cast<double>(levels - k + 1) * t_hoist +
                        static_cast<double>(k - 1) * t_decompose;
    if (cost < plan.cost) {
      plan.cost = cost;
      plan.k = k;
    }
  }
  return plan;
}

inline HoistPlan fixed_plan(HoistMode mode, std::size_t n) {  // distance.cpp:181-197
  const std::size_t levels = require_width_levels(n);
  HoistPlan plan;
  plan.n = n;
  if (mode == HoistMode::off) return plan;
  if (mode == HoistMode::full) {
    plan.k = levels + 1;
    return plan;
  }
  throw UsageError("dynamic plans come from plan_unfold with calibration");
}

inline std::vector<std::size_t> slot_reduce_steps(std::size_t n, std::size_t k) {
  if (n == 0 || (n & (n - 1))) throw WidthError("reduction width must be a power of two");
  if (k == 0) throw ParameterError("unfold factor starts at 1");
  std::size_t levels = 0;
  while ((std::size_t{1} << levels) < n) ++levels;
  const std::size_t unf = std::min(k - 1, levels);
  std::vector<std::size_t> s;
  for (std::size_t u = 1; u < (std::size_t{1} << unf); ++u) s.push_back(u);
  for (std::size_t j = unf; j < levels; ++j) s.push_back(std::size_t{1} << j);
  return s;
}

enum class SelectionRule { krum, multi_krum, median };
enum class DistanceMode { per_pair, row_sums };
struct DistanceOptions {
  bool lazy_relin = true;
  bool reduce_on_server = true;
};

// ================================================================== drop-in
// Host-side types with the reference's names and members (ckks.hpp:57-114,
// distance.hpp:31-38, 108-119, aggregation.hpp:77-82). A ciphertext's words
// are the LCLT payload order: [2][count][N] (c0 rows, then c1 rows).
struct Ciphertext {
  std::vector<std::uint64_t> words;
  std::size_t count = 0;  // live q-limbs = level + 1
  double scale = 0.0;
  int level() const { return static_cast<int>(count) - 1; }
  std::size_t size_bytes() const { return words.size() * sizeof(std::uint64_t); }
};

struct KeySwitchKey {  // [full digits][2][full+1][N], the reference's digit order
  std::vector<std::uint64_t> words;
};
struct RelinKey {
  KeySwitchKey key;
};
struct RotationKeySet {
  std::map<std::size_t, KeySwitchKey> steps;
  bool has_step(std::size_t step) const { return steps.count(step) != 0; }
};

struct PackedWeights {
  std::vector<Ciphertext> chunks;
  std::size_t dimension = 0;
  double prescale = 1.0;
  std::size_t chunk_count() const { return chunks.size(); }
};

struct SelectionMask {  // aggregation.hpp:77-82
  std::size_t n = 0;
  std::size_t l = 0;
  std::vector<Ciphertext> rank_rows;
  std::vector<Ciphertext> client_selectors;
};

struct EncryptedDistanceMatrix {  // distance.hpp:108-114
  DistanceMode mode = DistanceMode::per_pair;
  std::size_t n = 0;
  bool reduced = true;
  double value_scale = 1.0;
  std::map<std::pair<std::size_t, std::size_t>, Ciphertext> entries;
};

// ------------------------------------------------------------------ context
class CkksContext;

class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(lcl_context* ctx, std::size_t words) : ctx_(ctx), words_(words) {
    check(lcl_device_alloc(ctx, words * 8, &p_));
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept { *this = std::move(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(ctx_, o.ctx_);
    std::swap(p_, o.p_);
    std::swap(words_, o.words_);
    return *this;
  }
  ~DeviceBuffer() {
    if (p_) lcl_device_free(ctx_, p_);
  }
  std::uint64_t* data() const { return static_cast<std::uint64_t*>(p_); }
  std::size_t words() const { return words_; }
  void upload(const std::uint64_t* h) { check(lcl_copy_h2d(ctx_, p_, h, words_ * 8)); }
  std::vector<std::uint64_t> download() const {
    std::vector<std::uint64_t> h(words_);
    check(lcl_copy_d2h(ctx_, h.data(), p_, words_ * 8));
    return h;
  }

 private:
  lcl_context* ctx_ = nullptr;
  void* p_ = nullptr;
  std::size_t words_ = 0;
};

// All n clients' packed weights as one device batch [n][chunks][2][full][N]
// (the reference's std::vector<PackedWeights>, distance.hpp:31-38).
struct ClientBatch {
  DeviceBuffer words;
  std::size_t n = 0, chunks = 0, dimension = 0;
  double prescale = 1.0, scale = 0.0;
};

struct DeviceSelectionMask {  // aggregation.hpp:77-82 in HBM (client selectors only)
  DeviceBuffer client_selectors;  // [n][2][full][N]
  std::size_t n = 0, l = 0;
  double scale = 0.0;
};

struct DeviceDistanceMatrix {  // distance.hpp:108-114 in HBM, per_pair, (i<j) order
  DeviceBuffer entries;           // [pairs][2][full-1][N]
  std::size_t n = 0;
  bool reduced = true;
  double value_scale = 1.0, scale = 0.0;
};

struct PackedAggregate {  // PackedWeights returned by masked_aggregate
  DeviceBuffer chunks;    // [chunks][2][full-1 or full-2][N]
  std::size_t dimension = 0;
  double prescale = 1.0, scale = 0.0;
};

class CkksContext {
 public:
  explicit CkksContext(std::size_t degree, int depth = 3, bool secure = true, int device = 0) {
    check(lcl_context_create(degree, depth, secure ? 1 : 0, device, &h_));
    std::size_t full = 0;
    std::vector<std::uint64_t> p(depth + 2);
    check(lcl_context_primes(h_, p.data(), &full));
    full_ = full;
    primes_ = p;
    degree_ = degree;
  }
  CkksContext(const CkksContext&) = delete;
  CkksContext& operator=(const CkksContext&) = delete;
  ~CkksContext() { lcl_context_destroy(h_); }

  lcl_context* handle() const { return h_; }
  // every C-ABI call on this context goes through lock() (see "Threading")
  std::unique_lock<std::mutex> lock() const { return std::unique_lock<std::mutex>(mu_); }
  std::size_t degree() const { return degree_; }
  std::size_t slot_count() const { return degree_ / 2; }
  std::size_t prime_count() const { return full_; }
  const std::vector<std::uint64_t>& primes() const { return primes_; }
  std::size_t key_words() const { return full_ * 2 * (full_ + 1) * degree_; }

  void set_relin_key(const std::vector<std::uint64_t>& k) {
    auto g = lock();
    check(lcl_upload_relin_key(h_, k.data(), k.size()));
  }
  void set_rotation_key(std::size_t step, const std::vector<std::uint64_t>& k) {
    auto g = lock();
    check(lcl_upload_rotation_key(h_, step, k.data(), k.size()));
  }
  lcl_counts counters() const {
    auto g = lock();
    lcl_counts c;
    check(lcl_get_counts(h_, &c));
    return c;
  }
  void reset_counters() {
    auto g = lock();
    check(lcl_reset_counts(h_));
  }
  // CkksContext::serialize / deserialize (ckks.cpp:614-678), LCLT wire format
  std::vector<std::uint8_t> serialize(const Ciphertext& ct) const;
  Ciphertext deserialize(const std::uint8_t* data, std::size_t size) const;

 private:
  lcl_context* h_ = nullptr;
  std::size_t full_ = 0, degree_ = 0;
  std::vector<std::uint64_t> primes_;
  mutable std::mutex mu_;
};

// ------------------------------------------------------------------ hot path
inline DeviceDistanceMatrix build_distance_matrix(const CkksContext& ctx,
                                                  const ClientBatch& all,
                                                     const HoistPlan& plan,
                                                     const DistanceOptions& options = {}) {
  if (all.n < 2) throw ShapeError("pairwise distances need at least two clients");
  if (options.reduce_on_server) {
    const std::size_t needed = std::min(all.dimension, ctx.slot_count());
    std::size_t w = 1;
    while (w < needed) w <<= 1;
    if (plan.n < w) throw WidthError("plan width misses populated slots");
  }
  DeviceDistanceMatrix m;
  const std::size_t pairs = all.n * (all.n - 1) / 2;
  m.entries = DeviceBuffer(ctx.handle(), pairs * 2 * (ctx.prime_count() - 1) * ctx.degree());
  m.n = all.n;
  m.reduced = options.reduce_on_server;
  m.value_scale = all.prescale * all.prescale;
  auto g = ctx.lock();
  check(lcl_distance_matrix(ctx.handle(), all.words.data(), all.n, all.chunks, all.scale,
                            plan.n, plan.k, options.lazy_relin ? 1 : 0,
                            options.reduce_on_server ? 1 : 0, m.entries.data(), &m.scale));
  check(lcl_synchronize(ctx.handle()));
  return m;
}

inline PackedAggregate masked_aggregate(const CkksContext& ctx, const ClientBatch& weights,
                                        const DeviceSelectionMask& mask, SelectionRule rule) {
  if (weights.n == 0) throw ShapeError("no client weights to aggregate");
  if (weights.n != mask.n) throw ShapeError("mask rows do not match the client count");
  const bool average = rule == SelectionRule::multi_krum && mask.l > 1;
  const std::size_t m_out = ctx.prime_count() - (average ? 2 : 1);
  PackedAggregate out;
  out.chunks = DeviceBuffer(ctx.handle(), weights.chunks * 2 * m_out * ctx.degree());
  out.dimension = weights.dimension;
  out.prescale = weights.prescale;
  auto g = ctx.lock();
  check(lcl_masked_aggregate(ctx.handle(), weights.words.data(), mask.client_selectors.data(),
                             weights.n, weights.chunks, weights.scale, mask.scale, mask.l,
                             average ? 1 : 0, out.chunks.data(), &out.scale));
  check(lcl_synchronize(ctx.handle()));
  return out;
}

namespace detail {

// Keys stay resident on the device: a key is (re)uploaded only when the
// words behind it change identity (address or size) since the last call.
struct KeyCache {
  std::mutex mu;
  std::map<std::pair<lcl_context*, std::size_t>, std::pair<const void*, std::size_t>> up;
  static KeyCache& get() {
    static KeyCache c;
    return c;
  }
  // step 0 = the relinearisation key
  bool fresh(lcl_context* h, std::size_t step, const std::vector<std::uint64_t>& w) {
    std::lock_guard<std::mutex> g(mu);
    auto key = std::make_pair(h, step);
    auto val = std::make_pair(static_cast<const void*>(w.data()), w.size());
    auto it = up.find(key);
    if (it != up.end() && it->second == val) return true;
    up[key] = val;
    return false;
  }
};

inline void upload_keys(const CkksContext& ctx, const RelinKey& rk, const RotationKeySet* keys,
                        const std::vector<std::size_t>& steps) {
  KeyCache& kc = KeyCache::get();
  if (!kc.fresh(ctx.handle(), 0, rk.key.words))
    check(lcl_upload_relin_key(ctx.handle(), rk.key.words.data(), rk.key.words.size()));
  if (!keys) return;
  for (std::size_t raw : steps) {
    const std::size_t st = raw % ctx.slot_count();
    if (st == 0) continue;
    auto it = keys->steps.find(st);
    if (it == keys->steps.end()) throw KeyError("no rotation key for the requested step");
    if (!kc.fresh(ctx.handle(), st, it->second.words))
      check(lcl_upload_rotation_key(ctx.handle(), st, it->second.words.data(),
                                    it->second.words.size()));
  }
}

// [n][chunks][2][full][N] on the device from the host chunks (ShapeError on
// ragged or non-fresh input, AlignmentError on diverging scales).
inline DeviceBuffer gather(const CkksContext& ctx, const std::vector<PackedWeights>& all,
                           double* scale) {
  const std::size_t C = all.at(0).chunk_count();
  const std::size_t ctw = 2 * ctx.prime_count() * ctx.degree();
  DeviceBuffer d(ctx.handle(), all.size() * C * ctw);
  *scale = all[0].chunks.at(0).scale;
  for (std::size_t i = 0; i < all.size(); ++i) {
    const PackedWeights& pw = all[i];
    if (pw.chunk_count() != C || pw.dimension != all[0].dimension ||
        pw.prescale != all[0].prescale)
      throw ShapeError("packed weights disagree in length, chunking or prescale");
    for (std::size_t c = 0; c < C; ++c) {
      const Ciphertext& ct = pw.chunks[c];
      if (ct.count != ctx.prime_count() || ct.words.size() != ctw)
        throw ShapeError("client chunks must be fresh ciphertexts of the context");
      const double ref = std::max(std::fabs(ct.scale), std::fabs(*scale));
      if (std::fabs(ct.scale - *scale) > 1e-9 * ref) throw AlignmentError("operand scales diverge");
      check(lcl_copy_h2d(ctx.handle(), d.data() + (i * C + c) * ctw, ct.words.data(), ctw * 8));
    }
  }
  return d;
}

inline Ciphertext take(const std::vector<std::uint64_t>& h, std::size_t off, std::size_t count,
                       std::size_t N, double scale) {
  Ciphertext ct;
  ct.count = count;
  ct.scale = scale;
  ct.words.assign(h.begin() + off, h.begin() + off + 2 * count * N);
  return ct;
}

}  // namespace detail

// build_distance_matrix (distance.hpp:123-126), the reference's parameter
// list: per_pair or row_sums, lazy or eager, reduced on the server or left to
// the KGC. Bit-exact with the reference; one device round trip per call.
inline EncryptedDistanceMatrix build_distance_matrix(const CkksContext& ctx,
                                                const std::vector<PackedWeights>& all,
                                                const RelinKey& rk, const HoistPlan& plan,
                                                DistanceMode mode, const RotationKeySet& keys,
                                                const DistanceOptions& options) {
  const std::size_t n = all.size();
  if (n < 2) throw ShapeError("pairwise distances need at least two clients");
  if (options.reduce_on_server) {
    const std::size_t needed = std::min(all[0].dimension, ctx.slot_count());
    std::size_t w = 1;
    while (w < needed) w <<= 1;
    if (plan.n < w) throw WidthError("plan width misses populated slots");
  }
  auto g = ctx.lock();
  const std::vector<std::size_t> steps =
      options.reduce_on_server && plan.n > 1 ? slot_reduce_steps(plan.n, plan.k)
                                             : std::vector<std::size_t>{};
  detail::upload_keys(ctx, rk, &keys, steps);
  double in_scale = 0;
  const DeviceBuffer d = detail::gather(ctx, all, &in_scale);
  const std::size_t N = ctx.degree(), m = ctx.prime_count() - 1;
  const std::size_t pairs = n * (n - 1) / 2;
  const std::size_t entries = mode == DistanceMode::per_pair ? pairs : n;
  DeviceBuffer out(ctx.handle(), entries * 2 * m * N);
  double scale = 0;
  check(lcl_build_distance_matrix(ctx.handle(), d.data(), n, all[0].chunk_count(), in_scale,
                                  plan.n, plan.k, mode == DistanceMode::per_pair ? 0 : 1,
                                  options.lazy_relin ? 1 : 0, options.reduce_on_server ? 1 : 0,
                                  out.data(), &scale));
  check(lcl_synchronize(ctx.handle()));
  const std::vector<std::uint64_t> h = out.download();
  EncryptedDistanceMatrix res;
  res.mode = mode;
  res.n = n;
  res.reduced = options.reduce_on_server;
  res.value_scale = all[0].prescale * all[0].prescale;
  std::size_t e = 0;
  for (std::size_t i = 0; i < n; ++i) {
    if (mode == DistanceMode::row_sums) {
      res.entries.emplace(std::make_pair(i, i), detail::take(h, e++ * 2 * m * N, m, N, scale));
      continue;
    }
    for (std::size_t j = i + 1; j < n; ++j)
      res.entries.emplace(std::make_pair(i, j), detail::take(h, e++ * 2 * m * N, m, N, scale));
  }
  return res;
}

// masked_aggregate (aggregation.hpp:90-93), the reference's parameter list.
inline PackedWeights masked_aggregate(const CkksContext& ctx,
                                      const std::vector<PackedWeights>& weights,
                                      const SelectionMask& mask, SelectionRule rule,
                                      const RelinKey& rk) {
  if (weights.empty()) throw ShapeError("no client weights to aggregate");
  if (weights.size() != mask.n || mask.client_selectors.size() != mask.n)
    throw ShapeError("mask rows do not match the client count");
  auto g = ctx.lock();
  detail::upload_keys(ctx, rk, nullptr, {});
  double w_scale = 0;
  const DeviceBuffer d = detail::gather(ctx, weights, &w_scale);
  const std::size_t N = ctx.degree(), full = ctx.prime_count();
  const std::size_t ctw = 2 * full * N;
  DeviceBuffer sel(ctx.handle(), mask.n * ctw);
  for (std::size_t i = 0; i < mask.n; ++i) {
    const Ciphertext& s = mask.client_selectors[i];
    if (s.count != full || s.words.size() != ctw) throw ShapeError("selectors must be fresh ciphertexts");
    check(lcl_copy_h2d(ctx.handle(), sel.data() + i * ctw, s.words.data(), ctw * 8));
  }
  const bool average = rule == SelectionRule::multi_krum && mask.l > 1;
  const std::size_t mo = full - (average ? 2 : 1);
  const std::size_t C = weights[0].chunk_count();
  DeviceBuffer out(ctx.handle(), C * 2 * mo * N);
  double scale = 0;
  check(lcl_masked_aggregate(ctx.handle(), d.data(), sel.data(), weights.size(), C, w_scale,
                             mask.client_selectors[0].scale, mask.l, average ? 1 : 0, out.data(),
                             &scale));
  check(lcl_synchronize(ctx.handle()));
  const std::vector<std::uint64_t> h = out.download();
  PackedWeights res;
  res.dimension = weights[0].dimension;
  res.prescale = weights[0].prescale;
  for (std::size_t c = 0; c < C; ++c) res.chunks.push_back(detail::take(h, c * 2 * mo * N, mo, N, scale));
  return res;
}

// CkksContext::serialize / deserialize (ckks.cpp:614-678) over the LCLT wire format.
inline std::vector<std::uint8_t> CkksContext::serialize(const Ciphertext& ct) const {
  auto g = lock();
  DeviceBuffer d(h_, ct.words.size());
  d.upload(ct.words.data());
  std::vector<std::uint8_t> out(13 + ct.words.size() * 8);
  check(lcl_serialize(h_, d.data(), 1, ct.count, ct.scale, out.data(), out.size()));
  return out;
}

inline Ciphertext CkksContext::deserialize(const std::uint8_t* data, std::size_t size) const {
  auto g = lock();
  if (size < 13) throw DataError("not a ciphertext blob");
  const std::size_t count = std::min<std::size_t>(std::max<std::size_t>(data[12], 1), full_);
  DeviceBuffer d(h_, 2 * count * degree_);
  Ciphertext ct;
  check(lcl_deserialize(h_, data, size, size, 1, d.data(), &ct.scale));
  ct.count = count;
  ct.words = d.download();
  return ct;
}

}  // namespace lancelot_b200
