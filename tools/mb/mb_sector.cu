// mb_sector.cu -- microbenchmark (NOT the product path): random gathers at
// granule G bytes (8, 16, 32, 64, 128) per thread from a region of R bytes,
// written coalesced.  Index = hash(i) so no index stream is read.  Measures
// how the L1/L2/HBM path serves random requests by granule, to decide how
// the cfg5 gather should group its k1 loads (one 32-B sector per request vs
// one 8-B entry per request).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_sector mb_sector.cu
//   ./mb_sector  -> one JSON line per case
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}
struct V8 { uint32_t r[8]; };
__device__ __forceinline__ V8 ld256(const void* p) {
  V8 v;
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]),
                 "=r"(v.r[6]), "=r"(v.r[7]) : "l"(p));
  return v;
}
__device__ __forceinline__ void st256(void* p, const V8& v) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.r[0]), "r"(v.r[1]),
               "r"(v.r[2]), "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]), "r"(v.r[7]) : "memory");
}

// G = bytes per random block; each thread moves U blocks per iteration.
template <int G, int U>
__global__ void __launch_bounds__(256) gather(const char* __restrict__ src, uint64_t nblk_mask,
                                              char* __restrict__ dst, uint64_t count, uint32_t salt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < count; base += stride * U) {
    if constexpr (G == 8) {
      uint2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = base + u * stride;
        const uint64_t b = hash32(i ^ ((uint64_t)salt << 40)) & nblk_mask;
        v[u] = *(const uint2*)(src + b * 8);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs((uint2*)(dst) + base + u * stride, v[u]);
    } else if constexpr (G == 16) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = base + u * stride;
        const uint64_t b = hash32(i ^ ((uint64_t)salt << 40)) & nblk_mask;
        v[u] = *(const uint4*)(src + b * 16);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs((uint4*)(dst) + base + u * stride, v[u]);
    } else {
      constexpr int P = G / 32;
      V8 v[U][P];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = base + u * stride;
        const uint64_t b = hash32(i ^ ((uint64_t)salt << 40)) & nblk_mask;
#pragma unroll
        for (int p = 0; p < P; ++p) v[u][p] = ld256(src + b * G + 32 * p);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int p = 0; p < P; ++p) st256(dst + (base + u * stride) * G + 32 * p, v[u][p]);
    }
  }
}

// 8-B gathers whose 4 lanes-groups share a sector: lane l reads entry
// 4*hash(i/4) + (l & 3)  (in-warp coalescing of sector-mates).
template <int U>
__global__ void __launch_bounds__(256) gather_mates(const char* __restrict__ src, uint64_t nsec_mask,
                                                    char* __restrict__ dst, uint64_t count, uint32_t salt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < count; base += stride * U) {
    uint2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + u * stride;
      const uint64_t b = hash32((i >> 2) ^ ((uint64_t)salt << 40)) & nsec_mask;
      v[u] = *(const uint2*)(src + b * 32 + (i & 3) * 8);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs((uint2*)(dst) + base + u * stride, v[u]);
  }
}

__global__ void copyk(const uint4* __restrict__ s, uint4* __restrict__ d, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) __stcs(d + i, __ldcs(s + i));
}

template <typename F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f();
  cudaDeviceSynchronize();
  float best = 1e30f, tot = 0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    tot += ms; if (ms < best) best = ms;
  }
  return tot / reps;
}

int main() {
  const uint64_t SRC = 32ull << 30, OUT = 8ull << 30;
  char *src, *dst;
  if (cudaMalloc(&src, SRC) != cudaSuccess || cudaMalloc(&dst, OUT) != cudaSuccess) { printf("oom\n"); return 1; }
  cudaMemset(src, 1, SRC);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8;
  {
    float ms = timeit([&] { copyk<<<blocks, 256>>>((const uint4*)src, (uint4*)dst, OUT / 16); });
    printf("{\"case\":\"copy\",\"bytes\":%llu,\"ms\":%.3f,\"GBps\":%.1f}\n", (unsigned long long)OUT, ms, 2.0 * OUT / ms / 1e6);
  }
  const uint64_t regions[2] = {SRC, 64ull << 20};
  for (uint64_t R : regions) {
#define RUN(G, U)                                                                                   \
    {                                                                                               \
      const uint64_t count = OUT / G;                                                               \
      float ms = timeit([&] { gather<G, U><<<blocks, 256>>>(src, R / G - 1, dst, count, 7); });     \
      printf("{\"case\":\"gather\",\"G\":%d,\"U\":%d,\"region_MB\":%llu,\"ms\":%.3f,\"req_per_s\":%.3e,\"useful_GBps\":%.1f}\n", \
             G, U, (unsigned long long)(R >> 20), ms, count / ms * 1e3, 2.0 * OUT / ms / 1e6);       \
      fflush(stdout);                                                                               \
    }
    RUN(8, 8) RUN(8, 16) RUN(16, 8) RUN(32, 4) RUN(32, 8) RUN(64, 4) RUN(128, 2)
    {
      const uint64_t count = OUT / 8;
      float ms = timeit([&] { gather_mates<16><<<blocks, 256>>>(src, R / 32 - 1, dst, count, 7); });
      printf("{\"case\":\"gather_mates8\",\"region_MB\":%llu,\"ms\":%.3f,\"entries_per_s\":%.3e,\"useful_GBps\":%.1f}\n",
             (unsigned long long)(R >> 20), ms, count / ms * 1e3, 2.0 * OUT / ms / 1e6);
    }
  }
  return 0;
}
