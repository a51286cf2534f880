// mb_mlp.cu -- microbenchmark (NOT the product path): rate of random 8-byte
// gathers vs memory-level parallelism (loads in flight per thread U, CTAs of
// 256 threads per SM) for an L2-resident region (64 MB) and a 32 GiB one;
// with coalesced stores of the gathered values (as the step) or loads only.
// Decides whether the step's 2.16e11 entries/s is a latency/MLP limit
// (more warps or more loads in flight would raise it) or a throughput cap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_mlp mb_mlp.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}

template <int U, bool STORE>
__global__ void __launch_bounds__(256) gather8(const uint2* __restrict__ src, uint64_t mask,
                                               uint2* __restrict__ dst, uint64_t count, uint32_t* sink) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < count; base += stride * U) {
    uint2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[hash32(base + u * stride) & mask];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (STORE) __stcs(dst + base + u * stride, v[u]);
      else acc ^= v[u].x ^ v[u].y;
    }
  }
  if (!STORE && acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const uint64_t SRC = 32ull << 30, OUT = 8ull << 30, count = OUT / 8;
  uint2 *src, *dst;
  uint32_t* sink;
  if (cudaMalloc(&src, SRC) != cudaSuccess || cudaMalloc(&dst, OUT) != cudaSuccess ||
      cudaMalloc(&sink, 4) != cudaSuccess) {
    printf("oom\n");
    return 1;
  }
  cudaMemset(src, 1, SRC);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t regions[2] = {64ull << 20, SRC};
  for (uint64_t R : regions) {
    const uint64_t mask = R / 8 - 1;
#define RUN(U, ST, BPS)                                                                            \
    {                                                                                              \
      float best = 1e30f;                                                                          \
      for (int r = 0; r < 4; ++r) {                                                                \
        cudaEventRecord(a);                                                                        \
        gather8<U, ST><<<sms * BPS, 256>>>(src, mask, dst, count, sink);                           \
        cudaEventRecord(b);                                                                        \
        cudaEventSynchronize(b);                                                                   \
        float ms;                                                                                  \
        cudaEventElapsedTime(&ms, a, b);                                                           \
        if (r && ms < best) best = ms;                                                             \
      }                                                                                            \
      printf("{\"region_MB\": %llu, \"U\": %d, \"store\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, " \
             "\"req_per_s\": %.3e, \"err\": \"%s\"}\n", (unsigned long long)(R >> 20), U, (int)ST,   \
             BPS, best, count / (best * 1e-3), cudaGetErrorString(cudaGetLastError()));            \
      fflush(stdout);                                                                              \
    }
    RUN(8, true, 1) RUN(8, true, 2) RUN(8, true, 4) RUN(8, true, 8)
    RUN(16, true, 1) RUN(16, true, 2) RUN(16, true, 4) RUN(16, true, 8)
    RUN(32, true, 1) RUN(32, true, 2) RUN(32, true, 4)
    RUN(8, false, 8) RUN(16, false, 4) RUN(32, false, 2) RUN(32, false, 4)
  }
  return 0;
}
