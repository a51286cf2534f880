// qsim_kernels.cuh -- sm_100a kernels of the permutation-map hot path.
//
// Burger, arXiv quant-ph/0308158: each wiring-diagram step toggles the
// target address bit when all its control bits are 1 (P:L43 2(b)); the
// composite gather map is perm[i] = f_1(f_2(...f_n(i))) (readings R1, R2)
// and the state transform is k2[i] = k1[perm[i]].
//
// No tensor cores: there is no dense contraction.  Two walk algorithms:
//   * per-lane: one address per lane, 2 integer ops per gate (the direct
//     form of the step rule).
//   * bit-sliced: 32 addresses per thread held as 32 bit-plane words, one
//     word per address bit, in the thread's private shared-memory column.
//     A step is plane[t] ^= plane[c0] & plane[c1] (one logic op for 32
//     addresses); a 32x32 bit transpose turns planes back into addresses.
// Gathers move entries as raw 8/16-byte integers (bit-exact, R15).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qsim {

constexpr int kMaxGates = 4096;

// Gate list in the launch's kernel-parameter bank (constant bank 0): one
// 32-bit word per gate, kind | target << 8 | c0 << 16 | c1 << 24, with the
// unused control slots of NOT / CNOT normalised to 0 by the host.
template <int CAP>
struct GateList {
  uint32_t n;
  uint32_t w[CAP];
};

__device__ __forceinline__ uint32_t gate_kind(uint32_t w) { return w & 0xffu; }
__device__ __forceinline__ uint32_t gate_t(uint32_t w) { return (w >> 8) & 0xffu; }
__device__ __forceinline__ uint32_t gate_c0(uint32_t w) { return (w >> 16) & 0xffu; }
__device__ __forceinline__ uint32_t gate_c1(uint32_t w) { return w >> 24; }

// ---------------------------------------------------------------- loads/stores
__device__ __forceinline__ uint4 ld_stream_u4(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_gather(const uint2* p) { return __ldg(p); }
__device__ __forceinline__ uint4 ld_gather(const uint4* p) { return __ldg(p); }
__device__ __forceinline__ void st_stream(uint2* p, uint2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream_u32(uint32_t* p, uint32_t v) { __stcs(p, v); }

// ------------------------------------------------------------------ per-lane
// One address per lane: walk the gates last -> first, x ^= tmask when all
// control bits of x are set.  ADDR_PER_THREAD independent walks interleave
// to fill the ALU pipe.
template <int CAP, int MODE, typename T, int APT>
__global__ void __launch_bounds__(256)
k_walk_per_lane(const __grid_constant__ GateList<CAP> g, uint64_t start, uint64_t count,
                uint32_t* __restrict__ perm_out, const T* __restrict__ k1,
                T* __restrict__ k2_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * APT;
  for (uint64_t r0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * APT; r0 < count;
       r0 += stride) {
    uint32_t x[APT];
#pragma unroll
    for (int a = 0; a < APT; ++a) x[a] = (uint32_t)(start + r0 + a);
    for (int k = (int)g.n - 1; k >= 0; --k) {
      const uint32_t w = g.w[k];
      const uint32_t kind = gate_kind(w);
      const uint32_t cmask = (kind >= 1 ? (1u << gate_c0(w)) : 0u) |
                             (kind == 2 ? (1u << gate_c1(w)) : 0u);
      const uint32_t tmask = 1u << gate_t(w);
#pragma unroll
      for (int a = 0; a < APT; ++a)
        if ((~x[a] & cmask) == 0u) x[a] ^= tmask;
    }
#pragma unroll
    for (int a = 0; a < APT; ++a) {
      const uint64_t r = r0 + a;
      if (r < count) {
        if (MODE == 0) perm_out[r] = x[a];
        else k2_out[r] = ld_gather(k1 + x[a]);
      }
    }
  }
}

// ---------------------------------------------------------------- bit-sliced
// Tile = 1024 consecutive output addresses per warp.  Lane L, word bit l
// holds address tile*1024 + 32*l + L: address bits 0..4 are the lane
// (constant within a thread), bits 5..9 are the word bit l (the classic
// 0xAAAAAAAA.. patterns), bits >= 10 are the tile (constant per warp).
constexpr int kBsThreads = 256;
constexpr int kBsWarps = kBsThreads / 32;

// In-register 32x32 bit transpose: on return bit b of a[l] = bit l of the
// input a[b].  Five block-swap stages (16, 8, 4, 2, 1).
template <int J, uint32_t MASK>
__device__ __forceinline__ void transpose_stage(uint32_t (&a)[32]) {
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if ((k & J) == 0) {
      const uint32_t t = ((a[k] >> J) ^ a[k + J]) & MASK;
      a[k + J] ^= t;
      a[k] ^= t << J;
    }
  }
}

__device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
  transpose_stage<16, 0x0000ffffu>(a);
  transpose_stage<8, 0x00ff00ffu>(a);
  transpose_stage<4, 0x0f0f0f0fu>(a);
  transpose_stage<2, 0x33333333u>(a);
  transpose_stage<1, 0x55555555u>(a);
}

__device__ __forceinline__ uint32_t bs_init_plane(int b, uint32_t lane, uint64_t base) {
  if (b < 5) return ((lane >> b) & 1u) ? 0xffffffffu : 0u;
  if (b < 10) {
    const uint32_t pat[5] = {0xaaaaaaaau, 0xccccccccu, 0xf0f0f0f0u, 0xff00ff00u, 0xffff0000u};
    return pat[b - 5];
  }
  return ((base >> b) & 1u) ? 0xffffffffu : 0u;
}

template <int CAP, int MODE, typename T>
__global__ void __launch_bounds__(kBsThreads, 2)
k_walk_bitsliced(const __grid_constant__ GateList<CAP> g, uint64_t start, uint64_t end,
                 uint64_t tile_begin, uint64_t tile_end, uint32_t* __restrict__ perm_out,
                 const T* __restrict__ k1, T* __restrict__ k2_out) {
  __shared__ uint32_t S[32][kBsThreads];  // S[plane][thread]: private columns
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  for (uint64_t tile = tile_begin + (uint64_t)blockIdx.x * kBsWarps + warp; tile < tile_end;
       tile += (uint64_t)gridDim.x * kBsWarps) {
    const uint64_t base = tile << 10;
#pragma unroll
    for (int b = 0; b < 32; ++b) S[b][tid] = bs_init_plane(b, lane, base);
    // walk last -> first (R1, R2): one logic op per gate for 32 addresses
    for (int k = (int)g.n - 1; k >= 0; --k) {
      const uint32_t w = g.w[k];
      const uint32_t kind = gate_kind(w), t = gate_t(w);
      uint32_t x = S[t][tid];
      if (kind == 0) x = ~x;
      else if (kind == 1) x ^= S[gate_c0(w)][tid];
      else x ^= S[gate_c0(w)][tid] & S[gate_c1(w)][tid];
      S[t][tid] = x;
    }
    uint32_t a[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) a[b] = S[b][tid];
    transpose32(a);  // a[l] = perm(base + 32 l + lane)
    if (MODE == 0) {
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        const uint64_t addr = base + 32u * l + lane;
        if (addr >= start && addr < end) st_stream_u32(perm_out + (addr - start), a[l]);
      }
    } else {
      constexpr int B = 16;  // gathers in flight per thread
#pragma unroll
      for (int h = 0; h < 32; h += B) {
        T v[B];
#pragma unroll
        for (int l = 0; l < B; ++l) {
          const uint64_t addr = base + 32u * (h + l) + lane;
          if (addr >= start && addr < end) v[l] = ld_gather(k1 + a[h + l]);
        }
#pragma unroll
        for (int l = 0; l < B; ++l) {
          const uint64_t addr = base + 32u * (h + l) + lane;
          if (addr >= start && addr < end) st_stream(k2_out + (addr - start), v[l]);
        }
      }
    }
  }
}

// --------------------------------------------------------------------- apply
// k2[r] = k1[perm[r]]: perm streamed with 128-bit loads (4 indices), the
// gathers issued back to back (8 in flight per thread), k2 streamed out.
template <typename T>
__global__ void __launch_bounds__(256)
k_apply(const uint32_t* __restrict__ perm, uint64_t count, const T* __restrict__ k1,
        T* __restrict__ k2) {
  const uint64_t ngroups = count >> 2;  // groups of 4 entries
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; gi + nthreads < ngroups; gi += 2 * nthreads) {
    const uint4 p0 = ld_stream_u4(perm + 4 * gi);
    const uint4 p1 = ld_stream_u4(perm + 4 * (gi + nthreads));
    const T a0 = ld_gather(k1 + p0.x), a1 = ld_gather(k1 + p0.y);
    const T a2 = ld_gather(k1 + p0.z), a3 = ld_gather(k1 + p0.w);
    const T b0 = ld_gather(k1 + p1.x), b1 = ld_gather(k1 + p1.y);
    const T b2 = ld_gather(k1 + p1.z), b3 = ld_gather(k1 + p1.w);
    T* o0 = k2 + 4 * gi;
    T* o1 = k2 + 4 * (gi + nthreads);
    st_stream(o0 + 0, a0); st_stream(o0 + 1, a1); st_stream(o0 + 2, a2); st_stream(o0 + 3, a3);
    st_stream(o1 + 0, b0); st_stream(o1 + 1, b1); st_stream(o1 + 2, b2); st_stream(o1 + 3, b3);
  }
  if (gi < ngroups) {
    const uint4 p0 = ld_stream_u4(perm + 4 * gi);
    T* o0 = k2 + 4 * gi;
    st_stream(o0 + 0, ld_gather(k1 + p0.x)); st_stream(o0 + 1, ld_gather(k1 + p0.y));
    st_stream(o0 + 2, ld_gather(k1 + p0.z)); st_stream(o0 + 3, ld_gather(k1 + p0.w));
  }
  // ragged tail (count % 4 entries): first threads of block 0
  if (blockIdx.x == 0 && threadIdx.x < (count & 3u)) {
    const uint64_t r = (ngroups << 2) + threadIdx.x;
    k2[r] = ld_gather(k1 + perm[r]);
  }
}

}  // namespace qsim
