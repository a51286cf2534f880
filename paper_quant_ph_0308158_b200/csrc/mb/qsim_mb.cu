// qsim_mb.cu -- microbenchmark kernels (libqsim_mb.so; include/qsim_mb.h).
// Not on the product path: they measure the ceilings the product kernels are
// designed against (gather granularity and cache policy).
#include <cstdint>
#include <cuda_runtime.h>

#include "qsim_mb.h"

namespace {

template <int V>
__device__ __forceinline__ uint2 ld_var(const uint2* p) {
  uint2 r;
  if (V == 0) {
    r = __ldg(p);
  } else if (V == 1) {
    asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (V == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (V == 3) {
    asm volatile("ld.global.cs.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (V == 4) {
    asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (V == 5) {
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else if (V == 6) {
    asm volatile("ld.global.relaxed.gpu.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
  }
  return r;
}

template <int V, int U>
__global__ void __launch_bounds__(256)
k_mb_gather(const uint32_t* __restrict__ idx, uint64_t count, const uint2* __restrict__ k1,
            uint2* __restrict__ k2) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t groups = count / 4;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
       g += nthreads * U) {
    uint4 p[U];
    uint2 v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t gg = g + u * nthreads;
      if (gg < groups) p[u] = __ldcs(reinterpret_cast<const uint4*>(idx) + gg);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t gg = g + u * nthreads;
      if (gg < groups) {
        v[u][0] = ld_var<V>(k1 + p[u].x);
        v[u][1] = ld_var<V>(k1 + p[u].y);
        v[u][2] = ld_var<V>(k1 + p[u].z);
        v[u][3] = ld_var<V>(k1 + p[u].w);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t gg = g + u * nthreads;
      if (gg < groups) {
        uint4* o = reinterpret_cast<uint4*>(k2 + 4 * gg);
        __stcs(o, make_uint4(v[u][0].x, v[u][0].y, v[u][1].x, v[u][1].y));
        __stcs(o + 1, make_uint4(v[u][2].x, v[u][2].y, v[u][3].x, v[u][3].y));
      }
    }
  }
}

template <int V>
int launch(const uint32_t* idx, uint64_t count, const void* k1, void* k2, int unroll, int blocks,
           cudaStream_t st) {
  const uint2* a = static_cast<const uint2*>(k1);
  uint2* b = static_cast<uint2*>(k2);
  switch (unroll) {
    case 1: k_mb_gather<V, 1><<<blocks, 256, 0, st>>>(idx, count, a, b); break;
    case 2: k_mb_gather<V, 2><<<blocks, 256, 0, st>>>(idx, count, a, b); break;
    case 4: k_mb_gather<V, 4><<<blocks, 256, 0, st>>>(idx, count, a, b); break;
    default: return -1;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -6;
}

}  // namespace

extern "C" int qsim_mb_gather_c64(const uint32_t* idx, uint64_t count, const void* k1, void* k2,
                                  int32_t variant, int32_t unroll, int32_t blocks, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (blocks <= 0) blocks = 148 * 8;
  switch (variant) {
    case 0: return launch<0>(idx, count, k1, k2, unroll, blocks, st);
    case 1: return launch<1>(idx, count, k1, k2, unroll, blocks, st);
    case 2: return launch<2>(idx, count, k1, k2, unroll, blocks, st);
    case 3: return launch<3>(idx, count, k1, k2, unroll, blocks, st);
    case 4: return launch<4>(idx, count, k1, k2, unroll, blocks, st);
    case 5: return launch<5>(idx, count, k1, k2, unroll, blocks, st);
    case 6: return launch<6>(idx, count, k1, k2, unroll, blocks, st);
    case 7: return launch<7>(idx, count, k1, k2, unroll, blocks, st);
    default: return -1;
  }
}

// ---------------------------------------------------------------------------
// TMA tile::gather4 gather: k2[r] = k1[idx[r]] (complex64) with the k1 rows
// (16 bytes = the aligned pair holding the entry) fetched by the TMA engine
// into shared memory, 4 rows per instruction, STAGES-deep mbarrier ring.
// Warp 0 produces (each lane one gather4 per instruction), warps 1..4
// consume (select the 8-byte half, store k2 coalesced).
#include "qsim_tma.cuh"

namespace {

using namespace qsim;

template <int STAGES, int P, int kMbRows = 128 * P>
__global__ void __launch_bounds__(128 + 32 * P)
k_mb_tma_gather(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ idx,
                uint64_t count, uint2* __restrict__ k2) {
  extern __shared__ __align__(128) uint8_t smem[];
  // each gather4 (64 B) lands in its own 128-byte aligned slot
  uint4* buf = reinterpret_cast<uint4*>(smem);                       // [STAGES][kMbRows*2]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kMbRows * 32);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], P); mbar_init(&empty[s], 4 * 32); }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t nblocks = count / kMbRows;
  if (warp < P) {
    int s = 0; uint32_t ph = 0;
    for (uint64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
      mbar_wait(&empty[s], ph ^ 1u);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], kMbRows * 16 / P);
      __syncwarp();
      const uint4* ip = reinterpret_cast<const uint4*>(idx + b * kMbRows);
#pragma unroll
      for (int k = warp; k < kMbRows / 128; k += P) {
        const uint4 r = __ldg(ip + k * 32 + lane);
        tma_gather4(buf + s * kMbRows * 2 + (k * 32 + lane) * 8, &tm, &full[s], 0, (int)(r.x >> 1),
                    (int)(r.y >> 1), (int)(r.z >> 1), (int)(r.w >> 1));
      }
      if (++s == STAGES) { s = 0; ph ^= 1u; }
    }
  } else {
    const int t = threadIdx.x - 32 * P;   // 0..127
    int s = 0; uint32_t ph = 0;
    for (uint64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
      mbar_wait(&full[s], ph);
      const uint2* row = reinterpret_cast<const uint2*>(buf + s * kMbRows * 2);
#pragma unroll
      for (int k = 0; k < kMbRows / 128; ++k) {
        const int r = k * 128 + t;
        const uint32_t j = __ldg(idx + b * kMbRows + r);
        __stcs(k2 + b * kMbRows + r, row[(r >> 2) * 16 + (r & 3) * 2 + (j & 1u)]);
      }
      mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1u; }
    }
  }
}

}  // namespace

extern "C" int qsim_mb_tma_gather_c64(const uint32_t* idx, uint64_t count, const void* k1,
                                      uint64_t k1_entries, void* k2, int32_t stages,
                                      int32_t blocks, void* stream) {
  const int P = stages / 100;     // producer warps encoded in the hundreds
  stages %= 100;
  CUtensorMap tm;
  if (qsim::encode_row_map(&tm, k1, k1_entries / 2, 16) != 0) return -6;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (blocks <= 0) blocks = 148;
  const size_t sm = (size_t)stages * 128 * (P ? P : 1) * 32 + 2 * stages * 8;
#define QSIM_MB_ST(S, PP)                                                                      \
  case S * 100 + PP:                                                                            \
    cudaFuncSetAttribute(k_mb_tma_gather<S, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)sm);                                                             \
    k_mb_tma_gather<S, PP><<<blocks, 128 + 32 * PP, sm, st>>>(tm, idx, count,                 \
                                                              static_cast<uint2*>(k2));        \
    break;
  switch (stages * 100 + (P ? P : 1)) {
    QSIM_MB_ST(4, 4) QSIM_MB_ST(2, 8) QSIM_MB_ST(3, 8) QSIM_MB_ST(2, 16) QSIM_MB_ST(1, 16)
    QSIM_MB_ST(2, 12)
#undef QSIM_MB_ST
    default: return -1;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -6;
}

// ---------------------------------------------------------------------------
// Scatter: k2[idx[r]] = k1[r] (complex64), k1 streamed, k2 written at
// random positions -- the mirror image of the gather, to compare the cost of
// divergent stores with divergent loads.
namespace {
template <int U>
__global__ void __launch_bounds__(256)
k_mb_scatter(const uint32_t* __restrict__ idx, uint64_t count, const uint2* __restrict__ k1,
             uint2* __restrict__ k2) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += nthreads * U) {
    uint32_t d[U];
    uint2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t rr = r + u * nthreads;
      if (rr < count) { d[u] = __ldcs(idx + rr); v[u] = __ldcs(k1 + rr); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t rr = r + u * nthreads;
      if (rr < count) k2[d[u]] = v[u];
    }
  }
}
}  // namespace

extern "C" int qsim_mb_scatter_c64(const uint32_t* idx, uint64_t count, const void* k1, void* k2,
                                   int32_t unroll, int32_t blocks, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (blocks <= 0) blocks = 148 * 8;
  const uint2* a = static_cast<const uint2*>(k1);
  uint2* b = static_cast<uint2*>(k2);
  switch (unroll) {
    case 4: k_mb_scatter<4><<<blocks, 256, 0, st>>>(idx, count, a, b); break;
    case 8: k_mb_scatter<8><<<blocks, 256, 0, st>>>(idx, count, a, b); break;
    case 16: k_mb_scatter<16><<<blocks, 256, 0, st>>>(idx, count, a, b); break;
    default: return -1;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -6;
}
