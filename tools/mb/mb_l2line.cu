// mb_l2line.cu -- microbenchmark (NOT the product path): bandwidth of random
// whole-line reads that hit L2.  A region of R bytes (L2-resident when R is
// well under 126 MB) is read as random 128-byte lines, 8 lanes x 16 B per
// line (4 lines per warp instruction), U lines in flight per thread group.
// Decides whether a design that fetches every touched k1 line whole from L2
// (about 3.5x the k1 bytes through L2 at cfg5) can afford the L2 traffic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_l2line mb_l2line.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x *= 0x9e3779b97f4a7c15ull; x ^= x >> 29; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 32;
  return x;
}

template <int U>
__global__ void __launch_bounds__(256) lines(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                            uint64_t nline_mask, uint64_t iters) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t acc = 0;
  for (uint64_t it = 0; it < iters; ++it) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t line = mix((gw * iters + it) * (U * 4) + u * 4 + (lane >> 3)) & nline_mask;
      v[u] = __ldcg(src + line * 8 + (lane & 7));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x9e3779b9u) dst[0] = make_uint4(acc, 0, 0, 0);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4 *src, *dst;
  const size_t maxb = 4ull << 30;
  cudaMalloc(&src, maxb);
  cudaMalloc(&dst, 64);
  cudaMemset(src, 1, maxb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t R : {16ull << 20, 48ull << 20, 96ull << 20, 4ull << 30}) {
    const uint64_t nlines = R / 128;
    for (int bps : {4, 8}) {
      for (int U : {4, 8}) {
        const uint64_t warps = (uint64_t)sms * bps * 8;
        const uint64_t iters = 4096;
        const double bytes = (double)warps * iters * U * 4 * 128;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          if (U == 4) lines<4><<<sms * bps, 256>>>(src, dst, nlines - 1, iters);
          else lines<8><<<sms * bps, 256>>>(src, dst, nlines - 1, iters);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep && ms < best) best = ms;
        }
        printf("{\"region_MB\": %zu, \"ctas_per_sm\": %d, \"lines_in_flight_per_group\": %d, \"ms\": %.3f, "
               "\"GBps\": %.0f, \"lines_per_s\": %.3e, \"err\": \"%s\"}\n",
               R >> 20, bps, U, best, bytes / (best * 1e-3) / 1e9, bytes / 128 / (best * 1e-3),
               cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
      }
    }
  }
  return 0;
}
