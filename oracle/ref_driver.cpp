// ref_driver: test infrastructure only (never shipped, never on the product
// path). Links the UNMODIFIED reference core built by oracle/Makefile from
// /root/reference sources and drives it through its public API, mirroring the
// reference's own timing harness `measure_distance_phase`
// (proj/core/src/cli.cpp:308-350) and the server steps 3 and 8 of `run_round`
// (proj/core/src/protocol.cpp:430-432, 492-493).
//
//   ref_driver gen   <options> --out DIR   dump keys, inputs, outputs, counters
//   ref_driver bench <options> --reps R    time build_distance_matrix + masked_aggregate
//   ref_driver encrypt --N N --dim D       time pack_and_encrypt of one client
//   ref_driver keygen --N N --dim D --k K  time generate_keys (make_system's steps)
//   ref_driver ops   --N N --reps S        per-op latency (NTT, mult+relin+rescale,
//                                          hoisted rotations, rotate, decrypt_values), S s per op
//
//   ref_driver calibrate --N N --dim D --budget-mb B
//                                          calibrate() + plan_unfold (protocol.cpp:224-287)
//
// Options: --N --depth --clients --dim --k --seed --rule krum|multi_krum|median
//          --select i,j,... --secure 0|1 --lazy 0|1 --inter 0|1
//          --mode per_pair|row_sums --reduce 0|1 (DistanceMode / reduce_on_server)
//          --inputs encrypted|uniform  (uniform: client chunks and selectors are
//          uniform residues per row -- every evaluator op is data-oblivious, so
//          timing equals that of encrypted inputs without the ~10 min of
//          single-stream client encryption)
//          --k 0 --budget-mb B: the plan comes from calibrate() + plan_unfold
//          under a B MiB memory budget (HoistMode::dynamic_lp)
#include <algorithm>
#include <bit>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "lancelot/aggregation.hpp"
#include "lancelot/ckks.hpp"
#include "lancelot/distance.hpp"
#include "lancelot/threading.hpp"

using namespace lancelot;

namespace {

struct Opts {
  std::string cmd;
  std::size_t N = 256;
  int depth = 3;
  std::size_t clients = 4;
  std::size_t dim = 300;
  std::size_t k = 1;
  u64 seed = 1;
  std::string rule = "krum";
  std::vector<std::size_t> select{0};
  bool secure = false;
  bool lazy = true;
  bool inter = true;
  std::size_t reps = 3;
  std::string out = ".";
  std::string mode = "per_pair";
  bool reduce = true;
  bool uniform = false;
  double budget_mb = 1024.0;
};

Opts parse(int argc, char** argv) {
  Opts o;
  if (argc < 2) throw std::runtime_error("usage: ref_driver gen|bench [opts]");
  o.cmd = argv[1];
  for (int i = 2; i + 1 < argc; i += 2) {
    std::string k = argv[i], v = argv[i + 1];
    if (k == "--N") o.N = std::stoull(v);
    else if (k == "--depth") o.depth = std::stoi(v);
    else if (k == "--clients") o.clients = std::stoull(v);
    else if (k == "--dim") o.dim = std::stoull(v);
    else if (k == "--k") o.k = std::stoull(v);
    else if (k == "--seed") o.seed = std::stoull(v);
    else if (k == "--rule") o.rule = v;
    else if (k == "--secure") o.secure = v == "1";
    else if (k == "--lazy") o.lazy = v == "1";
    else if (k == "--inter") o.inter = v == "1";
    else if (k == "--reps") o.reps = std::stoull(v);
    else if (k == "--out") o.out = v;
    else if (k == "--mode") o.mode = v;
    else if (k == "--reduce") o.reduce = v == "1";
    else if (k == "--inputs") o.uniform = v == "uniform";
    else if (k == "--budget-mb") o.budget_mb = std::stod(v);
    else if (k == "--select") {
      o.select.clear();
      std::stringstream ss(v);
      std::string t;
      while (std::getline(ss, t, ',')) o.select.push_back(std::stoull(t));
    } else {
      throw std::runtime_error("unknown option " + k);
    }
  }
  return o;
}

void dump_poly(std::ofstream& f, const PolyRns& p) {
  for (std::size_t r = 0; r < p.row_count(); ++r) {
    f.write(reinterpret_cast<const char*>(p.row(r).data()),
            static_cast<std::streamsize>(p.row(r).size() * sizeof(u64)));
  }
}

void dump_ct(const std::string& path, const std::vector<const Ciphertext*>& cts) {
  std::ofstream f(path, std::ios::binary);
  for (const Ciphertext* c : cts) {
    dump_poly(f, c->c0);
    dump_poly(f, c->c1);
  }
}

void dump_ternary(const std::string& path, const TernaryCiphertext& t) {
  std::ofstream f(path, std::ios::binary);
  dump_poly(f, t.d0);
  dump_poly(f, t.d1);
  dump_poly(f, t.d2);
}

void dump_key(const std::string& path, const KeySwitchKey& k) {
  std::ofstream f(path, std::ios::binary);
  for (const auto& d : k.digits) {
    dump_poly(f, d.first);
    dump_poly(f, d.second);
  }
}

std::string counts_json(const OpCounts& c) {
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "{\"encryptions\": %llu, \"additions\": %llu, \"multiplications\": %llu, "
                "\"relinearizations\": %llu, \"rescales\": %llu, \"rotations\": %llu, "
                "\"mod_ups\": %llu}",
                (unsigned long long)c.encryptions, (unsigned long long)c.additions,
                (unsigned long long)c.multiplications,
                (unsigned long long)c.relinearizations,
                (unsigned long long)c.rescales, (unsigned long long)c.rotations,
                (unsigned long long)c.mod_ups);
  return buf;
}

std::string dbl(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

SelectionRule rule_of(const std::string& s) {
  if (s == "krum") return SelectionRule::krum;
  if (s == "multi_krum") return SelectionRule::multi_krum;
  if (s == "median") return SelectionRule::median;
  throw std::runtime_error("bad rule");
}

DistanceMode mode_of(const std::string& s) {
  if (s == "per_pair") return DistanceMode::per_pair;
  if (s == "row_sums") return DistanceMode::row_sums;
  throw std::runtime_error("bad mode");
}

// calibrate (protocol.cpp:224-253), restated over the public API because
// protocol.cpp (with the model / data / training stack) is not compiled
// into the checker: median of 11 hoisted_rotations({1}) and ({1, 2}) calls on
// a fresh encryption of 0.5 in every slot; t_hoist = t1, t_decompose =
// t2 - t1 (the reference's naming, see SURVEY "Reference defects").
struct Calib {
  double t_hoist, t_decompose, m_cipher;
};

Calib calibrate_ref(const CkksContext& ctx, const KeyBundle& keys, Sampler& rng) {
  std::vector<double> values(ctx.slot_count(), 0.5);
  const Ciphertext ct = ctx.encrypt(ctx.encode(values), keys.pk, rng);
  auto median_time = [&](const std::vector<std::size_t>& steps) {
    std::vector<double> times;
    for (int rep = 0; rep < 11; ++rep) {
      const auto a = std::chrono::steady_clock::now();
      (void)ctx.hoisted_rotations(ct, steps, keys.rotations);
      times.push_back(
          std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
    }
    std::sort(times.begin(), times.end());
    return times[times.size() / 2];
  };
  const double t1 = median_time({1});
  const double t2 = median_time({1, 2});
  return {std::max(t1, 1e-9), std::max(t2 - t1, 1e-9), (double)ct.size_bytes()};
}

// make_system's plan (protocol.cpp:255-287): dynamic_lp when k == 0 (tmp
// keys {1, 2} from derive_seed(seed, kTagTmpKeys)-like streams; any seed
// works: calibration only times), else fixed k.
HoistPlan make_plan(const CkksContext& ctx, const Opts& o, std::size_t width, Calib* cal) {
  if (o.k != 0) {
    HoistPlan plan = fixed_plan(HoistMode::off, width);
    plan.k = o.k;
    return plan;
  }
  Sampler tmp_rng(derive_seed(o.seed, 0x7A11u));
  const KeyBundle probe = ctx.generate_keys(tmp_rng, {1, 2});
  Sampler calib_rng(derive_seed(o.seed, 0xCA11u));
  const Calib c = calibrate_ref(ctx, probe, calib_rng);
  if (cal) *cal = c;
  return plan_unfold(c.t_hoist, c.t_decompose, c.m_cipher, o.budget_mb * 1048576.0, width);
}

struct System {
  std::unique_ptr<CkksContext> ctx;
  HoistPlan plan;
  Calib calib{0, 0, 0};
  KeyBundle keys;
  std::vector<std::size_t> steps;
  std::vector<PackedWeights> packed;
  SelectionMask mask;
};

System setup(const Opts& o) {
  System s;
  CkksParams p;
  p.ring_degree = o.N;
  p.depth = o.depth;
  p.security = o.secure ? SecurityLevel::bits128 : SecurityLevel::none;
  s.ctx = std::make_unique<CkksContext>(p);
  const CkksContext& ctx = *s.ctx;
  const std::size_t width = std::bit_ceil(std::min(o.dim, ctx.slot_count()));
  // make_system (protocol.cpp:255-287): a fixed unfold factor, or the
  // calibrated plan; no rotation keys when slot sums are left to the KGC.
  s.plan = make_plan(ctx, o, width, &s.calib);
  s.steps = o.reduce ? slot_reduce_steps(width, s.plan.k) : std::vector<std::size_t>{};
  if (s.steps.size() > 512) throw CapacityError("unfold plan needs more than 512 rotation keys");
  Sampler key_rng(derive_seed(o.seed, 5));
  s.keys = ctx.generate_keys(key_rng, s.steps);
  // measure_distance_phase input generation (cli.cpp:316-329).
  Sampler rng(derive_seed(o.seed, 0xAB1A7Eu));
  s.packed.resize(o.clients);
  if (o.uniform) {
    const std::size_t C = chunk_count_for(o.dim, ctx.slot_count());
    // one Sampler per client, filled on worker threads (setup only)
    s.mask.n = o.clients;
    s.mask.l = o.select.size();
    s.mask.client_selectors.resize(o.clients);
    parallel_for(o.clients, [&](std::size_t i) {
      Sampler crng(derive_seed(o.seed, 0xAB1A7Eu + 1 + i));
      auto uniform_ct = [&]() {
        Ciphertext c;
        c.c0 = PolyRns(ctx.basis(), ctx.basis()->prime_count(), false, Domain::evaluation);
        c.c1 = c.c0;
        crng.uniform_poly(c.c0);
        crng.uniform_poly(c.c1);
        c.scale = ctx.scale();
        return c;
      };
      s.packed[i].dimension = o.dim;
      s.packed[i].prescale = 1.0;
      s.packed[i].chunks.reserve(C);
      for (std::size_t ch = 0; ch < C; ++ch) s.packed[i].chunks.push_back(uniform_ct());
      s.mask.client_selectors[i] = uniform_ct();
    });
    return s;
  }
  for (std::size_t i = 0; i < o.clients; ++i) {
    std::vector<double> w(o.dim);
    for (double& x : w) x = rng.uniform_real() - 0.5;
    s.packed[i] = pack_and_encrypt(ctx, w, s.keys.pk, rng);
  }
  SelectionResult sel{rule_of(o.rule), o.select, o.select.size()};
  Sampler mask_rng(derive_seed(o.seed, 0x3000000000000000ull));
  s.mask = build_mask(ctx, sel, o.clients, s.keys.pk, mask_rng);
  return s;
}

int cmd_gen(const Opts& o) {
  System s = setup(o);
  const CkksContext& ctx = *s.ctx;
  const std::string d = o.out;
  {
    std::ofstream f(d + "/sk.bin", std::ios::binary);
    dump_poly(f, s.keys.sk.s);
  }
  dump_key(d + "/relin.bin", s.keys.relin.key);
  for (const auto& [step, key] : s.keys.rotations.steps) {
    dump_key(d + "/rot_" + std::to_string(step) + ".bin", key);
  }
  for (std::size_t i = 0; i < o.clients; ++i) {
    std::vector<const Ciphertext*> v;
    for (const auto& c : s.packed[i].chunks) v.push_back(&c);
    dump_ct(d + "/client_" + std::to_string(i) + ".bin", v);
    dump_ct(d + "/sel_" + std::to_string(i) + ".bin", {&s.mask.client_selectors[i]});
  }

  DistanceOptions dopt;
  dopt.lazy_relin = o.lazy;
  dopt.reduce_on_server = o.reduce;
  ctx.counters().reset();
  const EncryptedDistanceMatrix m =
      build_distance_matrix(ctx, s.packed, s.keys.relin, s.plan,
                            mode_of(o.mode), s.keys.rotations, dopt);
  const OpCounts dist_ops = ctx.counters().snapshot();
  ctx.counters().reset();
  const PackedWeights agg =
      masked_aggregate(ctx, s.packed, s.mask, rule_of(o.rule), s.keys.relin);
  const OpCounts agg_ops = ctx.counters().snapshot();

  std::ostringstream js;
  js << "{\n";
  const RnsBasis& b = *ctx.basis();
  js << "  \"N\": " << o.N << ", \"depth\": " << o.depth << ", \"slots\": "
     << ctx.slot_count() << ",\n";
  js << "  \"primes\": [";
  for (std::size_t i = 0; i < b.prime_count(); ++i) js << (i ? ", " : "") << b.prime(i).value;
  js << "], \"special\": " << b.special().value << ",\n";
  js << "  \"psi\": [";
  for (std::size_t i = 0; i <= b.prime_count(); ++i)
    js << (i ? ", " : "") << b.tables_or_special(i).psi;
  js << "],\n";
  js << "  \"mode\": \"" << o.mode << "\", \"reduced\": " << (m.reduced ? "true" : "false")
     << ", \"value_scale\": " << dbl(m.value_scale) << ",\n";
  js << "  \"width\": " << s.plan.n << ", \"k\": " << s.plan.k << ", \"steps\": [";
  for (std::size_t i = 0; i < s.steps.size(); ++i) js << (i ? ", " : "") << s.steps[i];
  js << "],\n  \"rot_keys\": [";
  {
    bool first = true;
    for (const auto& [step, key] : s.keys.rotations.steps) {
      js << (first ? "" : ", ") << step;
      first = false;
    }
  }
  js << "],\n";
  js << "  \"chunks\": " << s.packed[0].chunk_count() << ", \"client_scale\": "
     << dbl(s.packed[0].chunks[0].scale) << ", \"client_level\": "
     << s.packed[0].chunks[0].level() << ",\n";
  js << "  \"dist_ops\": " << counts_json(dist_ops) << ",\n";
  js << "  \"agg_ops\": " << counts_json(agg_ops) << ",\n";

  // Outputs.
  js << "  \"dist\": [";
  bool first = true;
  for (const auto& [key, ct] : m.entries) {
    dump_ct(d + "/dist_" + std::to_string(key.first) + "_" + std::to_string(key.second) + ".bin",
            {&ct});
    const auto slots = ctx.decrypt_values(ct, s.keys.sk);
    js << (first ? "" : ", ") << "{\"i\": " << key.first << ", \"j\": " << key.second
       << ", \"level\": " << ct.level() << ", \"scale\": " << dbl(ct.scale)
       << ", \"slot0\": " << dbl(slots[0]) << "}";
    first = false;
  }
  js << "],\n";
  {
    // the LCLT wire bytes (CkksContext::serialize) of client 0's first chunk
    // and of the first matrix entry, for the ingest parity tests
    const auto b0 = ctx.serialize(s.packed[0].chunks[0]);
    std::ofstream(d + "/lclt_client_0_0.bin", std::ios::binary)
        .write(reinterpret_cast<const char*>(b0.data()), (std::streamsize)b0.size());
    const auto b1 = ctx.serialize(m.entries.begin()->second);
    std::ofstream(d + "/lclt_dist_first.bin", std::ios::binary)
        .write(reinterpret_cast<const char*>(b1.data()), (std::streamsize)b1.size());
  }
  {
    std::vector<const Ciphertext*> v;
    for (const auto& c : agg.chunks) v.push_back(&c);
    dump_ct(d + "/agg.bin", v);
    const std::vector<double> w = decrypt_weights(ctx, agg, s.keys.sk);
    js << "  \"agg_level\": " << agg.chunks[0].level() << ", \"agg_scale\": "
       << dbl(agg.chunks[0].scale) << ", \"agg_head\": [";
    for (std::size_t i = 0; i < std::min<std::size_t>(8, w.size()); ++i)
      js << (i ? ", " : "") << dbl(w[i]);
    js << "],\n";
  }
  // Plaintext oracle for the distances (cli input generation replayed).
  {
    Sampler rng(derive_seed(o.seed, 0xAB1A7Eu));
    std::vector<std::vector<double>> ws(o.clients);
    // Replay is not possible without re-encrypting (the stream is shared), so
    // the plaintext weights are recovered by decryption instead.
    js << "  \"plain_dist\": [";
    for (std::size_t i = 0; i < o.clients; ++i) ws[i] = decrypt_weights(ctx, s.packed[i], s.keys.sk);
    bool f2 = true;
    for (std::size_t i = 0; i < o.clients; ++i)
      for (std::size_t j = i + 1; j < o.clients; ++j) {
        double acc = 0;
        for (std::size_t t = 0; t < o.dim; ++t) acc += (ws[i][t] - ws[j][t]) * (ws[i][t] - ws[j][t]);
        js << (f2 ? "" : ", ") << dbl(acc);
        f2 = false;
      }
    js << "]";
  }

  if (o.inter) {
    // Intermediates of pair (0,1): the lazy ternary accumulator, relin, rescale
    // and every hoisted / iterative rotation of slot_reduce.
    const PackedWeights& a = s.packed[0];
    const PackedWeights& bb = s.packed[1];
    TernaryCiphertext acc = ctx.hsquare(ctx.hsub(a.chunks[0], bb.chunks[0]));
    for (std::size_t c = 1; c < a.chunk_count(); ++c)
      ctx.lazy_accumulate(acc, ctx.hsquare(ctx.hsub(a.chunks[c], bb.chunks[c])));
    dump_ternary(d + "/p01_acc.bin", acc);
    const Ciphertext rl = ctx.relinearize(acc, s.keys.relin);
    dump_ct(d + "/p01_relin.bin", {&rl});
    const Ciphertext rs = ctx.rescale(rl);
    dump_ct(d + "/p01_rescale.bin", {&rs});
    // Each rotation key applied once to the rescaled ciphertext.
    for (const auto& [step, key] : s.keys.rotations.steps) {
      const Ciphertext r = ctx.rotate(rs, step, s.keys.rotations);
      dump_ct(d + "/p01_rot_" + std::to_string(step) + ".bin", {&r});
    }
    // Aggregate chunk 0 pieces.
    TernaryCiphertext t = ctx.hmult_triple(s.packed[0].chunks[0], s.mask.client_selectors[0]);
    for (std::size_t i = 1; i < o.clients; ++i)
      ctx.lazy_accumulate(t, ctx.hmult_triple(s.packed[i].chunks[0], s.mask.client_selectors[i]));
    dump_ternary(d + "/agg0_acc.bin", t);
  }
  js << "\n}\n";
  std::ofstream(d + "/meta.json") << js.str();
  return 0;
}

int cmd_bench(const Opts& o) {
  const auto t0 = std::chrono::steady_clock::now();
  System s = setup(o);
  const double setup_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const CkksContext& ctx = *s.ctx;
  DistanceOptions dopt;
  dopt.lazy_relin = o.lazy;
  dopt.reduce_on_server = o.reduce;
  std::printf("{\"setup_s\": %.3f, \"threads\": %zu, \"k\": %zu, \"t_hoist\": %.6g, "
              "\"t_decompose\": %.6g, \"m_cipher\": %.0f, \"reps\": [",
              setup_s, worker_count(), s.plan.k, s.calib.t_hoist, s.calib.t_decompose,
              s.calib.m_cipher);
  for (std::size_t r = 0; r < o.reps; ++r) {
    const auto a = std::chrono::steady_clock::now();
    const EncryptedDistanceMatrix m =
        build_distance_matrix(ctx, s.packed, s.keys.relin, s.plan,
                              mode_of(o.mode), s.keys.rotations, dopt);
    const auto b = std::chrono::steady_clock::now();
    const PackedWeights agg =
        masked_aggregate(ctx, s.packed, s.mask, rule_of(o.rule), s.keys.relin);
    const auto c = std::chrono::steady_clock::now();
    std::printf("%s{\"distance_s\": %.6f, \"aggregate_s\": %.6f}", r ? ", " : "",
                std::chrono::duration<double>(b - a).count(),
                std::chrono::duration<double>(c - b).count());
    std::fflush(stdout);
    (void)m;
    (void)agg;
  }
  std::printf("]}\n");
  return 0;
}

// Per-op latency of the reference evaluator at ring degree N, on the shapes
// of its own google-benchmark harness (proj/benchmarks/bench_ring.cpp:28-165,
// BM_NttRoundtrip / BM_MultRelinRescale / BM_RotationsHoisted(7) /
// BM_Rotate): a fresh ciphertext at full level, keys for steps 1..7 and the
// powers of two. Each op repeats until ~budget seconds have elapsed (>= 2 reps).
int cmd_ops(const Opts& o) {
  CkksParams p;
  p.ring_degree = o.N;
  p.depth = o.depth;
  p.security = o.secure ? SecurityLevel::bits128 : SecurityLevel::none;
  const CkksContext ctx(p);
  std::vector<std::size_t> steps = {1, 2, 3, 4, 5, 6, 7};
  for (std::size_t st = 8; st < ctx.slot_count(); st *= 2) steps.push_back(st);
  Sampler key_rng(101);
  const KeyBundle keys = ctx.generate_keys(key_rng, steps);
  Sampler rng(202);
  std::vector<double> v(ctx.slot_count());
  for (double& x : v) x = rng.uniform_real() - 0.5;
  const Ciphertext ct = ctx.encrypt(ctx.encode(v), keys.pk, rng);
  const double budget = (double)o.reps;  // seconds per op
  auto time_op = [&](auto&& f) {
    std::size_t n = 0;
    const auto a = std::chrono::steady_clock::now();
    double el = 0;
    do {
      f();
      ++n;
      el = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
    } while (el < budget || n < 2);
    return el / (double)n;
  };
  PolyRns poly = ct.c0;
  const double ntt = time_op([&] {
    poly.ntt_inverse();
    poly.ntt_forward();
  });
  const double mrr = time_op([&] {
    const Ciphertext out = ctx.rescale(ctx.relinearize(ctx.hsquare(ct), keys.relin));
    (void)out;
  });
  const std::vector<std::size_t> h7 = {1, 2, 3, 4, 5, 6, 7};
  const double hoist = time_op([&] {
    const std::vector<Ciphertext> out = ctx.hoisted_rotations(ct, h7, keys.rotations);
    (void)out;
  });
  const double rot = time_op([&] {
    const Ciphertext out = ctx.rotate(ct, 1, keys.rotations);
    (void)out;
  });
  const double dec = time_op([&] {  // BM_Decrypt
    const std::vector<double> vals = ctx.decrypt_values(ct, keys.sk);
    (void)vals;
  });
  std::printf("{\"N\": %zu, \"limbs\": %zu, \"threads\": %zu, \"ntt_roundtrip_s\": %.9f, "
              "\"mult_relin_rescale_s\": %.9f, \"hoisted7_s\": %.9f, \"rotate_s\": %.9f, "
              "\"decrypt_values_s\": %.9f}\n",
              o.N, ct.c0.row_count(), worker_count(), ntt, mrr, hoist, rot, dec);
  return 0;
}

// pack_and_encrypt of one client's weight vector (dim uniform_real - 0.5
// draws, as measure_distance_phase draws them), timed on this thread.
int cmd_encrypt(const Opts& o) {
  CkksParams p;
  p.ring_degree = o.N;
  p.depth = o.depth;
  p.security = o.secure ? SecurityLevel::bits128 : SecurityLevel::none;
  const CkksContext ctx(p);
  Sampler key_rng(derive_seed(o.seed, 5));
  const KeyBundle keys = ctx.generate_keys(key_rng, {});
  Sampler rng(derive_seed(o.seed, 0xAB1A7Eu));
  std::vector<double> w(o.dim);
  for (double& x : w) x = rng.uniform_real() - 0.5;
  const auto a = std::chrono::steady_clock::now();
  const PackedWeights pw = pack_and_encrypt(ctx, w, keys.pk, rng);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  std::printf("{\"N\": %zu, \"dim\": %zu, \"chunks\": %zu, \"pack_and_encrypt_s\": %.6f}\n", o.N,
              o.dim, pw.chunk_count(), s);
  return 0;
}

// generate_keys for slot_reduce_steps(bit_ceil(min(dim, slots)), k), as
// make_system does (protocol.cpp:277-285), timed on this thread.
int cmd_keygen(const Opts& o) {
  CkksParams p;
  p.ring_degree = o.N;
  p.depth = o.depth;
  p.security = o.secure ? SecurityLevel::bits128 : SecurityLevel::none;
  const CkksContext ctx(p);
  const std::size_t width = std::bit_ceil(std::min(o.dim, ctx.slot_count()));
  const std::vector<std::size_t> steps = slot_reduce_steps(width, o.k);
  Sampler key_rng(derive_seed(o.seed, 5));
  const auto a = std::chrono::steady_clock::now();
  const KeyBundle kb = ctx.generate_keys(key_rng, steps);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  std::printf("{\"N\": %zu, \"rotation_keys\": %zu, \"generate_keys_s\": %.6f}\n", o.N,
              kb.rotations.steps.size(), s);
  return 0;
}

// calibrate() + plan_unfold for ring degree N and a dim-parameter model
// (make_system with HoistMode::dynamic_lp, protocol.cpp:255-287).
int cmd_calibrate(const Opts& o) {
  CkksParams p;
  p.ring_degree = o.N;
  p.depth = o.depth;
  p.security = o.secure ? SecurityLevel::bits128 : SecurityLevel::none;
  const CkksContext ctx(p);
  const std::size_t width = std::bit_ceil(std::min(o.dim, ctx.slot_count()));
  Opts d = o;
  d.k = 0;
  Calib c{0, 0, 0};
  const HoistPlan plan = make_plan(ctx, d, width, &c);
  std::printf("{\"N\": %zu, \"width\": %zu, \"t_hoist\": %.9g, \"t_decompose\": %.9g, "
              "\"m_cipher\": %.0f, \"budget_mb\": %g, \"k\": %zu, \"cost\": %.9g, "
              "\"keys\": %zu}\n",
              o.N, width, c.t_hoist, c.t_decompose, c.m_cipher, o.budget_mb, plan.k, plan.cost,
              slot_reduce_steps(width, plan.k).size());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Opts o = parse(argc, argv);
    if (o.cmd == "gen") return cmd_gen(o);
    if (o.cmd == "bench") return cmd_bench(o);
    if (o.cmd == "ops") return cmd_ops(o);
    if (o.cmd == "encrypt") return cmd_encrypt(o);
    if (o.cmd == "keygen") return cmd_keygen(o);
    if (o.cmd == "calibrate") return cmd_calibrate(o);
    std::fprintf(stderr, "unknown command %s\n", o.cmd.c_str());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
