// lancelot_b200.hpp — C++ mirror of the reference's server API over the C-ABI.
//
// For C++ callers of the reference (lancelot::core, /root/reference/proj/core)
// this header keeps the names, argument meaning and exception types of
//   build_distance_matrix   distance.hpp:123-126
//   masked_aggregate        aggregation.hpp:90-93
//   HoistPlan / slot_reduce_steps / fixed_plan       distance.hpp:67-99
//   errors                  errors.hpp:27-104
// while the work runs on the B200 through include/lancelot_b200.h. Ciphertext
// batches live in HBM (DeviceBuffer); the layouts are the reference's
// (limb-major u64, c0 rows then c1 rows).
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
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
struct HoistPlan {  // distance.hpp:70-78 (the cost-model fields are host-only)
  std::size_t k = 1;
  std::size_t n = 1;
};

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

struct SelectionMask {  // aggregation.hpp:77-82 (client selectors only)
  DeviceBuffer client_selectors;  // [n][2][full][N]
  std::size_t n = 0, l = 0;
  double scale = 0.0;
};

struct EncryptedDistanceMatrix {  // distance.hpp:108-114, per_pair, (i<j) order
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
  std::size_t degree() const { return degree_; }
  std::size_t slot_count() const { return degree_ / 2; }
  std::size_t prime_count() const { return full_; }
  const std::vector<std::uint64_t>& primes() const { return primes_; }
  std::size_t key_words() const { return full_ * 2 * (full_ + 1) * degree_; }

  void set_relin_key(const std::vector<std::uint64_t>& k) {
    check(lcl_upload_relin_key(h_, k.data(), k.size()));
  }
  void set_rotation_key(std::size_t step, const std::vector<std::uint64_t>& k) {
    check(lcl_upload_rotation_key(h_, step, k.data(), k.size()));
  }
  lcl_counts counters() const {
    lcl_counts c;
    check(lcl_get_counts(h_, &c));
    return c;
  }
  void reset_counters() { check(lcl_reset_counts(h_)); }

 private:
  lcl_context* h_ = nullptr;
  std::size_t full_ = 0, degree_ = 0;
  std::vector<std::uint64_t> primes_;
};

// ------------------------------------------------------------------ hot path
inline EncryptedDistanceMatrix build_distance_matrix(const CkksContext& ctx,
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
  EncryptedDistanceMatrix m;
  const std::size_t pairs = all.n * (all.n - 1) / 2;
  m.entries = DeviceBuffer(ctx.handle(), pairs * 2 * (ctx.prime_count() - 1) * ctx.degree());
  m.n = all.n;
  m.reduced = options.reduce_on_server;
  m.value_scale = all.prescale * all.prescale;
  check(lcl_distance_matrix(ctx.handle(), all.words.data(), all.n, all.chunks, all.scale,
                            plan.n, plan.k, options.lazy_relin ? 1 : 0,
                            options.reduce_on_server ? 1 : 0, m.entries.data(), &m.scale));
  check(lcl_synchronize(ctx.handle()));
  return m;
}

inline PackedAggregate masked_aggregate(const CkksContext& ctx, const ClientBatch& weights,
                                        const SelectionMask& mask, SelectionRule rule) {
  if (weights.n == 0) throw ShapeError("no client weights to aggregate");
  if (weights.n != mask.n) throw ShapeError("mask rows do not match the client count");
  const bool average = rule == SelectionRule::multi_krum && mask.l > 1;
  const std::size_t m_out = ctx.prime_count() - (average ? 2 : 1);
  PackedAggregate out;
  out.chunks = DeviceBuffer(ctx.handle(), weights.chunks * 2 * m_out * ctx.degree());
  out.dimension = weights.dimension;
  out.prescale = weights.prescale;
  check(lcl_masked_aggregate(ctx.handle(), weights.words.data(), mask.client_selectors.data(),
                             weights.n, weights.chunks, weights.scale, mask.scale, mask.l,
                             average ? 1 : 0, out.chunks.data(), &out.scale));
  check(lcl_synchronize(ctx.handle()));
  return out;
}

}  // namespace lancelot_b200
