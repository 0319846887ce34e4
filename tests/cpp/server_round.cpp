// Drives the C++ mirror (include/lancelot_b200.hpp) the way the reference's
// own server does: run_round's steps 3 and 8 (protocol.cpp:419-432, 480-499)
// written against the mirror with the reference's types, member names and
// call expressions -- received LCLT bytes deserialized chunk by chunk, then
// build_distance_matrix(ctx, received, server.evk, server.plan, server.mode,
// server.rotations, server.options) and masked_aggregate(ctx, received,
// mask, rule, server.evk). The static_asserts pin the exact parameter lists
// of distance.hpp:123-126 and aggregation.hpp:90-93. Inputs / outputs are raw
// u64 files written / checked by tests/test_cpp_mirror.py.
//   server_round DIR N n chunks dim width k rule(0 krum,1 multi_krum) l scale
//                [mode(0 per_pair,1 row_sums) reduce(0|1)]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "lancelot_b200.hpp"

namespace L = lancelot_b200;

// distance.hpp:123-126 and aggregation.hpp:90-93, parameter for parameter
using BuildDistanceMatrix = L::EncryptedDistanceMatrix (*)(
    const L::CkksContext&, const std::vector<L::PackedWeights>&, const L::RelinKey&,
    const L::HoistPlan&, L::DistanceMode, const L::RotationKeySet&, const L::DistanceOptions&);
using MaskedAggregate = L::PackedWeights (*)(const L::CkksContext&,
                                             const std::vector<L::PackedWeights>&,
                                             const L::SelectionMask&, L::SelectionRule,
                                             const L::RelinKey&);
static_assert(std::is_same_v<decltype(static_cast<BuildDistanceMatrix>(&L::build_distance_matrix)),
                             BuildDistanceMatrix>);
static_assert(std::is_same_v<decltype(static_cast<MaskedAggregate>(&L::masked_aggregate)),
                             MaskedAggregate>);
// the reference's HoistPlan field order (distance.hpp:70-78)
static_assert(offsetof(L::HoistPlan, k) < offsetof(L::HoistPlan, t_hoist) &&
              offsetof(L::HoistPlan, m_budget) < offsetof(L::HoistPlan, n) &&
              offsetof(L::HoistPlan, n) < offsetof(L::HoistPlan, cost));

// protocol.hpp:208-216, the members run_round reads
struct ServerState {
  L::RelinKey evk;
  L::RotationKeySet rotations;
  L::HoistPlan plan;
  L::DistanceOptions options;
  L::DistanceMode mode = L::DistanceMode::per_pair;
  std::vector<L::PackedWeights> received;
};

static std::vector<std::uint64_t> slurp(const std::string& p) {
  std::ifstream f(p, std::ios::binary | std::ios::ate);
  if (!f) throw std::runtime_error("missing " + p);
  const std::size_t bytes = f.tellg();
  f.seekg(0);
  std::vector<std::uint64_t> v(bytes / 8);
  f.read(reinterpret_cast<char*>(v.data()), bytes);
  return v;
}

static void dump(const std::string& p, const std::vector<std::uint64_t>& v) {
  std::ofstream(p, std::ios::binary).write(reinterpret_cast<const char*>(v.data()), v.size() * 8);
}

int main(int argc, char** argv) {
  if (argc != 11 && argc != 13) {
    std::fprintf(stderr, "usage: server_round DIR N n chunks dim width k rule l scale [mode reduce]\n");
    return 2;
  }
  const std::string d = argv[1];
  const std::size_t N = std::stoull(argv[2]), n = std::stoull(argv[3]), C = std::stoull(argv[4]);
  const std::size_t dim = std::stoull(argv[5]), width = std::stoull(argv[6]), k = std::stoull(argv[7]);
  const int rule_i = std::atoi(argv[8]);
  const std::size_t l = std::stoull(argv[9]);
  const double scale = std::atof(argv[10]);
  const bool row_sums = argc == 13 && std::atoi(argv[11]) == 1;
  const bool reduce = argc != 13 || std::atoi(argv[12]) == 1;
  try {
    const L::CkksContext ctx(N, 3, false, 0);
    const std::size_t full = ctx.prime_count();
    const std::size_t ctw = 2 * full * N;
    ServerState server;
    server.evk.key.words = slurp(d + "/relin.bin");
    server.plan = L::fixed_plan(L::HoistMode::off, width);
    server.plan.k = k;
    server.mode = row_sums ? L::DistanceMode::row_sums : L::DistanceMode::per_pair;
    server.options.reduce_on_server = reduce;
    if (reduce)
      for (std::size_t s : L::slot_reduce_steps(width, k))
        server.rotations.steps[s].words = slurp(d + "/rot_" + std::to_string(s) + ".bin");
    // the clients' messages: LCLT bytes per chunk (ctx.serialize on the
    // client side), rebuilt by the server exactly as protocol.cpp:419-429
    const std::vector<std::uint64_t> words = slurp(d + "/clients.bin");
    std::vector<std::vector<std::vector<std::uint8_t>>> msgs(n);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t c = 0; c < C; ++c) {
        L::Ciphertext ct;
        ct.count = full;
        ct.scale = scale;
        ct.words.assign(words.begin() + (i * C + c) * ctw, words.begin() + (i * C + c + 1) * ctw);
        msgs[i].push_back(ctx.serialize(ct));
      }
    std::vector<L::PackedWeights> received(n);
    for (std::size_t i = 0; i < n; ++i) {
      L::PackedWeights pw;
      pw.dimension = dim;
      pw.prescale = 1.0;
      pw.chunks.reserve(msgs[i].size());
      for (const auto& bytes : msgs[i]) pw.chunks.push_back(ctx.deserialize(bytes.data(), bytes.size()));
      received[i] = std::move(pw);
    }
    const std::vector<std::uint64_t> sw = slurp(d + "/selectors.bin");
    L::SelectionMask mask;
    mask.n = n;
    mask.l = l;
    for (std::size_t i = 0; i < n; ++i) {
      L::Ciphertext ct;
      ct.count = full;
      ct.scale = scale;
      ct.words.assign(sw.begin() + i * ctw, sw.begin() + (i + 1) * ctw);
      const std::vector<std::uint8_t> bytes = ctx.serialize(ct);
      mask.client_selectors.push_back(ctx.deserialize(bytes.data(), bytes.size()));
    }
    const L::SelectionRule rule = rule_i == 1 ? L::SelectionRule::multi_krum : L::SelectionRule::krum;
    const_cast<L::CkksContext&>(ctx).reset_counters();

    // run_round step 3 (protocol.cpp:430-432) and step 8 (:492-493), verbatim
    L::EncryptedDistanceMatrix matrix =
        build_distance_matrix(ctx, received, server.evk, server.plan,
                              server.mode, server.rotations, server.options);
    const L::PackedWeights aggregated =
        masked_aggregate(ctx, received, mask, rule, server.evk);
    const lcl_counts c = ctx.counters();

    std::vector<std::uint64_t> out;
    double dist_scale = 0;
    for (const auto& [key, ct] : matrix.entries) {
      out.insert(out.end(), ct.words.begin(), ct.words.end());
      dist_scale = ct.scale;
    }
    dump(d + "/out_dist.bin", out);
    out.clear();
    for (const L::Ciphertext& ct : aggregated.chunks) out.insert(out.end(), ct.words.begin(), ct.words.end());
    dump(d + "/out_agg.bin", out);

    // a const context shared by threads, as the reference allows: calls are
    // serialised by the mirror, results identical
    L::EncryptedDistanceMatrix again[2];
    std::thread t0([&] { again[0] = build_distance_matrix(ctx, received, server.evk, server.plan,
                                                          server.mode, server.rotations, server.options); });
    std::thread t1([&] { again[1] = build_distance_matrix(ctx, received, server.evk, server.plan,
                                                          server.mode, server.rotations, server.options); });
    t0.join();
    t1.join();
    bool same = true;
    for (int t = 0; t < 2; ++t)
      for (const auto& [key, ct] : matrix.entries) same = same && again[t].entries.at(key).words == ct.words;

    std::printf("{\"dist_scale\": %.17g, \"agg_scale\": %.17g, \"entries\": %zu, \"reduced\": %d, "
                "\"threads_identical\": %d, \"additions\": %llu, \"multiplications\": %llu, "
                "\"relinearizations\": %llu, \"rescales\": %llu, \"rotations\": %llu, "
                "\"mod_ups\": %llu}\n",
                dist_scale, aggregated.chunks.at(0).scale, matrix.entries.size(),
                matrix.reduced ? 1 : 0, same ? 1 : 0, (unsigned long long)c.additions,
                (unsigned long long)c.multiplications, (unsigned long long)c.relinearizations,
                (unsigned long long)c.rescales, (unsigned long long)c.rotations,
                (unsigned long long)c.mod_ups);
    // exception parity: too narrow a plan is a WidthError, a missing key a
    // KeyError, a corrupted blob a DataError
    try {
      L::HoistPlan narrow = server.plan;
      narrow.n = width / 2;
      if (reduce) {
        build_distance_matrix(ctx, received, server.evk, narrow, server.mode, server.rotations,
                              server.options);
        std::printf("no-throw\n");
        return 1;
      }
    } catch (const L::WidthError&) {
    }
    if (reduce && width > 1) {
      try {
        L::RotationKeySet missing = server.rotations;
        missing.steps.erase(missing.steps.begin());
        build_distance_matrix(ctx, received, server.evk, server.plan, server.mode, missing,
                              server.options);
        std::printf("no-throw\n");
        return 1;
      } catch (const L::KeyError&) {
      }
    }
    try {
      std::vector<std::uint8_t> bad = msgs[0][0];
      bad[0] = 'X';
      ctx.deserialize(bad.data(), bad.size());
      std::printf("no-throw\n");
      return 1;
    } catch (const L::DataError&) {
    }
    // the device-resident variant gives the same words
    if (!row_sums && reduce) {
      L::ClientBatch all;
      all.words = L::DeviceBuffer(ctx.handle(), n * C * ctw);
      all.words.upload(words.data());
      all.n = n;
      all.chunks = C;
      all.dimension = dim;
      all.scale = scale;
      const L::DeviceDistanceMatrix dm = L::build_distance_matrix(ctx, all, server.plan);
      std::vector<std::uint64_t> flat;
      for (const auto& [key, ct] : matrix.entries) flat.insert(flat.end(), ct.words.begin(), ct.words.end());
      if (dm.entries.download() != flat) {
        std::printf("device-resident variant differs\n");
        return 1;
      }
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
