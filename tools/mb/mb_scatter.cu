// mb_scatter.cu -- microbenchmark (NOT the product path): random BLOCK reads
// with sequential writes (a gather, as the step reads k1) against sequential
// reads with random block writes (a scatter), each block moved exactly once
// (a bijection on block indices), 32 GiB -> 32 GiB.  Decides whether a
// traversal that reads k1 in order and writes k2 at random lines could beat
// the gather's DRAM rate.  16-B chunks, 8 lanes per 128-B line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_scatter mb_scatter.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// bijection on the low `bits` bits
__device__ __forceinline__ uint64_t mix(uint64_t x, int bits) {
  const uint64_t m = (bits == 64) ? ~0ull : ((1ull << bits) - 1);
  x = (x * 0x9e3779b97f4a7c15ull) & m;
  x ^= x >> (bits / 2);
  x = (x * 0xbf58476d1ce4e5b9ull) & m;
  x ^= x >> (bits / 3);
  x = (x * 0x94d049bb133111ebull) & m;
  return x;
}

// B = block bytes (multiple of 16); chunk c of block b
template <int B, bool SCATTER>
__global__ void __launch_bounds__(256) move(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                            uint64_t nchunks, int blk_bits) {
  constexpr int CPB = B / 16;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nchunks; i += stride) {
    const uint64_t blk = i / CPB, c = i % CPB;
    const uint64_t r = mix(blk, blk_bits) * CPB + c;
    if (SCATTER) __stcs(dst + r, __ldcs(src + i));
    else __stcs(dst + i, src[r]);
  }
}

// read-only: random blocks, each read once, XOR-reduced (a store only if the
// impossible value shows up)
template <int B>
__global__ void __launch_bounds__(256) readonly(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                uint64_t nchunks, int blk_bits) {
  constexpr int CPB = B / 16;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nchunks; i += stride) {
    const uint64_t blk = i / CPB, c = i % CPB;
    const uint4 v = src[mix(blk, blk_bits) * CPB + c];
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x9e3779b9u) dst[0] = make_uint4(acc, 0, 0, 0);
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const uint64_t BYTES = 32ull << 30, n = BYTES / 16;
  uint4 *src, *dst;
  if (cudaMalloc(&src, BYTES) != cudaSuccess || cudaMalloc(&dst, BYTES) != cudaSuccess) {
    printf("oom\n");
    return 1;
  }
  cudaMemset(src, 1, BYTES);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned grid = sms * 8;
  auto rep = [&](const char* name, int B, float ms) {
    printf("{\"case\": \"%s\", \"block_B\": %d, \"ms\": %.3f, \"GBps_moved\": %.0f, \"GBps_dram\": %.0f, \"err\": \"%s\"}\n",
           name, B, ms, BYTES / (ms * 1e-3) / 1e9, 2.0 * BYTES / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
#define CASE(BB)                                                                                   \
  {                                                                                                \
    int bits = 0;                                                                                  \
    while ((1ull << bits) < BYTES / BB) ++bits;                                                    \
    rep("gather", BB, timeit([&] { move<BB, false><<<grid, 256>>>(src, dst, n, bits); }));        \
    rep("scatter", BB, timeit([&] { move<BB, true><<<grid, 256>>>(src, dst, n, bits); }));         \
    { float ms = timeit([&] { readonly<BB><<<grid, 256>>>(src, dst, n, bits); });                  \
      printf("{\"case\": \"readonly\", \"block_B\": %d, \"ms\": %.3f, \"GBps_read\": %.0f}\n", BB, ms, \
             BYTES / (ms * 1e-3) / 1e9); }                                                          \
  }
  CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512) CASE(2048) CASE(8192)
  return 0;
}
