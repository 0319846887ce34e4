// Is the aggregate tensor / small-pair accumulation held back by the
// power-of-two strides of the client layout ([n][C][2][m][N] u64: poly rows
// 2 MiB apart, chunks 4 MiB apart at N = 2^16, m = 4)? Streams the cfg3
// client volume (20 clients x 342 chunks) with the aggregate kernel's access
// pattern (a thread reads its 16-byte slot pair of poly 0 and poly 1 of one
// chunk for every client, cp.async ring, 256 threads) and with the pair
// kernel's (a CTA copies 64-byte pieces of both polys of all 20 clients per
// chunk, 32 threads), once with the dense pitch and once with a padded chunk
// pitch (+pad bytes per chunk). Prints GB/s of each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 stride_probe.cu -o stride_probe && ./stride_probe
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
typedef uint64_t u64;
typedef uint32_t u32;

__device__ __forceinline__ void cp16(void* s, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// aggregate-like: thread = 2 slots of one limb row of one chunk; walks clients
template <int ST>
__global__ void __launch_bounds__(256) agg_like(const u64* __restrict__ c, u32 n, u32 chunks,
                                                u64 chunk_pitch, u32 slots, u64* sink) {
  extern __shared__ ulonglong2 ring[];
  const u32 ch = blockIdx.x % chunks;
  const u32 e = ((blockIdx.x / chunks) * blockDim.x + threadIdx.x) * 2;
  const u64* w = c + (u64)ch * chunk_pitch + e;
  const u64 cs = (u64)chunks * chunk_pitch;
  ulonglong2* my = ring + threadIdx.x;
  auto issue = [&](u32 i, u32 s) {
    if (i < n) {
      cp16(my + (2 * s) * blockDim.x, w + (u64)i * cs);
      cp16(my + (2 * s + 1) * blockDim.x, w + (u64)i * cs + slots);
    }
    commit();
  };
  for (int s = 0; s < ST - 1; ++s) issue(s, s);
  u64 acc = 0;
  u32 st = 0;
  for (u32 i = 0; i < n; ++i) {
    wait<ST - 2>();
    const ulonglong2 a = my[(2 * st) * blockDim.x], b = my[(2 * st + 1) * blockDim.x];
    issue(i + ST - 1, st == 0 ? ST - 1 : st - 1);
    acc ^= a.x ^ a.y ^ b.x ^ b.y;
    st = st + 1 == ST ? 0 : st + 1;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

// pair-like: CTA = TS-slot tile of one limb row (the pair kernel: TS = 8);
// per chunk copies TS * 8 bytes of both polys of all n clients into a ring
// stage; one barrier per chunk
template <int ST, int TS>
__global__ void __launch_bounds__(128) pair_like(const u64* __restrict__ c, u32 n, u32 chunks,
                                                u64 chunk_pitch, u32 slots, u64* sink) {
  extern __shared__ u64 tile[];  // [ST][n][2][TS]
  const u32 a0 = blockIdx.x * TS;
  const u64 cs = (u64)chunks * chunk_pitch;
  const u32 tw = n * 2 * TS;
  constexpr u32 VP = TS / 2;  // 16-byte vectors per poly piece
  auto issue = [&](u32 ch, u32 s) {
    if (ch < chunks)
      for (u32 v = threadIdx.x; v < n * 2 * VP; v += blockDim.x) {
        const u32 cl = v / (2 * VP), h = (v / VP) % 2, q = (v % VP) * 2;
        cp16(tile + s * tw + cl * 2 * TS + h * TS + q,
             c + (u64)cl * cs + (u64)ch * chunk_pitch + (u64)h * slots + a0 + q);
      }
    commit();
  };
  for (int s = 0; s < ST - 1; ++s) issue(s, s);
  u64 acc = 0;
  u32 st = 0;
  for (u32 ch = 0; ch < chunks; ++ch) {
    wait<ST - 2>();
    __syncthreads();
    issue(ch + ST - 1, st == 0 ? ST - 1 : st - 1);
    for (u32 k = threadIdx.x; k < tw; k += blockDim.x) acc ^= tile[st * tw + k];
    st = st + 1 == ST ? 0 : st + 1;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

template <int ST, int TS>
void run_pair(const u64* c, u32 n, u32 chunks, u64 pitch, u32 slots, u64* sink, u32 threads, double bytes) {
  const size_t sm = (size_t)ST * n * 2 * TS * 8;
  cudaFuncSetAttribute(pair_like<ST, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    pair_like<ST, TS><<<slots / TS, threads, sm>>>(c, n, chunks, pitch, slots, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r) best = ms < best ? ms : best;
  }
  printf("  pair-like ST=%2d TS=%2d (%3u thr, %4zu B/stage-client-poly): %.3f ms  %.0f GB/s\n", ST, TS, threads,
         (size_t)TS * 8, best, bytes / best / 1e6);
}

int main() {
  const u32 n = 20, chunks = 342, N = 1 << 16, m = 4;
  const u32 slots = m * N;                 // one poly: m limb rows
  const u64 ct = 2ull * slots;             // words per chunk (dense pitch)
  const u64 pads[] = {0, 512};     // extra words per chunk
  u64* sink;
  cudaMalloc(&sink, 8);
  for (u64 pad : pads) {
    const u64 pitch = ct + pad;
    const u64 words = (u64)n * chunks * pitch;
    u64* c = nullptr;
    if (cudaMalloc(&c, words * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(c, 1, words * 8);
    const double bytes = (double)n * chunks * ct * 8;  // what is read
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    {
      constexpr int ST = 6;
      const size_t sm = ST * 2 * 256 * 16;
      cudaFuncSetAttribute(agg_like<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      const u32 grid = slots / 2 / 256 * chunks;
      float best = 1e9f;
      for (int r = 0; r < 4; ++r) {
        cudaEventRecord(a);
        agg_like<ST><<<grid, 256, sm>>>(c, n, chunks, pitch, slots, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = ms < best ? ms : best;
      }
      printf("pad %4llu words  aggregate-like: %.3f ms  %.0f GB/s\n", (unsigned long long)pad, best, bytes / best / 1e6);
    }
    if (pad == 0) {
      run_pair<6, 8>(c, n, chunks, pitch, slots, sink, 32, bytes);
      run_pair<6, 8>(c, n, chunks, pitch, slots, sink, 64, bytes);
      run_pair<12, 8>(c, n, chunks, pitch, slots, sink, 32, bytes);
      run_pair<6, 16>(c, n, chunks, pitch, slots, sink, 64, bytes);
      run_pair<6, 32>(c, n, chunks, pitch, slots, sink, 128, bytes);
      run_pair<4, 32>(c, n, chunks, pitch, slots, sink, 128, bytes);
    } else {
      run_pair<6, 8>(c, n, chunks, pitch, slots, sink, 32, bytes);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaFree(c);
  }
  return 0;
}
