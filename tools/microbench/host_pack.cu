// Can host-side bit packing of LCLT payloads (u64 residues < 2^40 / 2^44)
// outrun PCIe? Measures (a) H2D of the u64 words from pinned memory, (b) T
// host threads packing 40-bit fields, (c) the pipelined pack -> H2D of the
// packed stream (chunked ring), all over the same pinned input.
//   nvcc -O3 -Xcompiler -O3,-pthread host_pack.cu -o host_pack && ./host_pack [GB] [threads]
#include <cuda_runtime.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
typedef uint64_t u64;
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
// 8 words of 40 bits -> 5 u64
static inline void pack40(const u64* __restrict in, u64* __restrict out, size_t n8) {
  for (size_t g = 0; g < n8; ++g) {
    const u64* a = in + 8 * g;
    u64* o = out + 5 * g;
    o[0] = a[0] | (a[1] << 40);
    o[1] = (a[1] >> 24) | (a[2] << 16) | (a[3] << 56);
    o[2] = (a[3] >> 8) | (a[4] << 32);
    o[3] = (a[4] >> 32) | (a[5] << 8) | (a[6] << 48);
    o[4] = (a[6] >> 16) | (a[7] << 24);
  }
}
int main(int argc, char** argv) {
  double gb = argc > 1 ? atof(argv[1]) : 8.0;
  int T = argc > 2 ? atoi(argv[2]) : (int)std::thread::hardware_concurrency();
  size_t words = (size_t)(gb * 1e9 / 8) / 4096 * 4096;
  u64 *src, *pk, *d;
  cudaMallocHost(&src, words * 8);
  cudaMallocHost(&pk, words * 5);
  cudaMalloc(&d, words * 8);
  for (size_t i = 0; i < words; ++i) src[i] = (i * 0x9E3779B97F4A7C15ull) & ((1ull << 40) - 1);
  memset(pk, 0, words * 5);
  cudaStream_t s;
  cudaStreamCreate(&s);
  // (a) H2D of u64 words
  for (int r = 0; r < 2; ++r) {
    double t0 = now();
    cudaMemcpyAsync(d, src, words * 8, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    double t = now() - t0;
    printf("(a) H2D u64 %.2f GB: %.3f s = %.1f GB/s\n", words * 8 / 1e9, t, words * 8 / 1e9 / t);
  }
  // (b) pack with T threads
  for (int r = 0; r < 2; ++r) {
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        size_t a = words / 8 * t / T, b = words / 8 * (t + 1) / T;
        pack40(src + 8 * a, pk + 5 * a, b - a);
      });
    for (auto& x : th) x.join();
    double t = now() - t0;
    printf("(b) pack %d threads: %.3f s = %.1f GB/s of u64 input\n", T, t, words * 8 / 1e9 / t);
  }
  // (c) pipelined: chunks of CH words; threads pack chunk k, main thread issues H2D of chunk k when packed
  const size_t CH = 1 << 24;  // 16 M words = 128 MB input, 80 MB packed
  const size_t nch = words / CH;
  for (int r = 0; r < 2; ++r) {
    double t0 = now();
    for (size_t k = 0; k < nch; ++k) {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          size_t a = CH / 8 * t / T, b = CH / 8 * (t + 1) / T;
          pack40(src + k * CH + 8 * a, pk + (k * CH + 8 * a) * 5 / 8, b - a);
        });
      for (auto& x : th) x.join();
      cudaMemcpyAsync((char*)d + k * CH * 5, (char*)pk + k * CH * 5, CH * 5, cudaMemcpyHostToDevice, s);
    }
    cudaStreamSynchronize(s);
    double t = now() - t0;
    printf("(c) pack+H2D pipelined: %.3f s = %.1f GB/s of u64 input (%zu chunks)\n", t, nch * CH * 8 / 1e9 / t, nch);
  }
  return 0;
}
