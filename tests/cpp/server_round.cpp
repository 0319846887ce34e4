// Drives the C++ mirror (include/lancelot_b200.hpp) the way a reference
// caller would: keys + client batch + mask in, distance matrix + aggregate
// out. Inputs / outputs are raw u64 files written / checked by
// tests/test_cpp_mirror.py.
//   server_round DIR N n chunks dim width k rule(0 krum,1 multi_krum) l scale
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "lancelot_b200.hpp"

namespace L = lancelot_b200;

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
  if (argc != 11) {
    std::fprintf(stderr, "usage: server_round DIR N n chunks dim width k rule l scale\n");
    return 2;
  }
  const std::string d = argv[1];
  const std::size_t N = std::stoull(argv[2]), n = std::stoull(argv[3]), C = std::stoull(argv[4]);
  const std::size_t dim = std::stoull(argv[5]), width = std::stoull(argv[6]), k = std::stoull(argv[7]);
  const int rule = std::atoi(argv[8]);
  const std::size_t l = std::stoull(argv[9]);
  const double scale = std::atof(argv[10]);
  try {
    L::CkksContext ctx(N, 3, false, 0);
    ctx.set_relin_key(slurp(d + "/relin.bin"));
    for (std::size_t s : L::slot_reduce_steps(width, k)) ctx.set_rotation_key(s, slurp(d + "/rot_" + std::to_string(s) + ".bin"));
    L::ClientBatch all;
    all.words = L::DeviceBuffer(ctx.handle(), n * C * 2 * ctx.prime_count() * N);
    all.words.upload(slurp(d + "/clients.bin").data());
    all.n = n;
    all.chunks = C;
    all.dimension = dim;
    all.scale = scale;
    L::SelectionMask mask;
    mask.client_selectors = L::DeviceBuffer(ctx.handle(), n * 2 * ctx.prime_count() * N);
    mask.client_selectors.upload(slurp(d + "/selectors.bin").data());
    mask.n = n;
    mask.l = l;
    mask.scale = scale;
    ctx.reset_counters();
    const L::EncryptedDistanceMatrix m = L::build_distance_matrix(ctx, all, L::HoistPlan{k, width});
    const L::PackedAggregate a = L::masked_aggregate(
        ctx, all, mask, rule == 1 ? L::SelectionRule::multi_krum : L::SelectionRule::krum);
    dump(d + "/out_dist.bin", m.entries.download());
    dump(d + "/out_agg.bin", a.chunks.download());
    const lcl_counts c = ctx.counters();
    std::printf("{\"dist_scale\": %.17g, \"agg_scale\": %.17g, \"rotations\": %llu}\n", m.scale,
                a.scale, (unsigned long long)c.rotations);
    // exception parity: too narrow a plan is a WidthError
    try {
      L::build_distance_matrix(ctx, all, L::HoistPlan{k, width / 2});
      std::printf("no-throw\n");
      return 1;
    } catch (const L::WidthError&) {
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
