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
//
// Traversal order: "counter" c runs over [0, 2^M); the output it handles is
// sigma(c), a permutation of the address bits (identity = natural order).
// sigma fixes bits 0..2 (0..1 for complex128), so every warp store covers
// whole 32-byte sectors; the lanes' output bits are lo = sigma(lane).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qsim {

constexpr int kMaxGates = 4096;
constexpr uint32_t kOnesPlane = 32;  // bit-sliced: an all-ones plane (absent control)
constexpr uint32_t kSignPlane = 33;  // bit-sliced: the row-value (sign) plane

// Gate kinds (include/qsim.h): 0 NOT, 1 CNOT, 2 CCNOT toggle the target when
// the controls are 1; 3 Z, 4 CZ, 5 CCZ put -1 on the rows whose
// target and controls are 1 (phased permutations, reading R17); 6 SWAP
// exchanges bits target and c0.
// Bit-sliced ops: 0 toggle, 1 swap, 2 phase.
constexpr uint32_t kOpToggle = 0, kOpSwap = 1, kOpPhase = 2;

// Gate list in the launch's kernel-parameter bank (constant bank 0), one
// 32-bit word per gate.  Per-lane format: kind | target << 8 | c0 << 16 |
// c1 << 24 (unused controls 0).  Bit-sliced format: target | c0 << 8 |
// c1 << 16 | op << 24 with absent controls = kOnesPlane.
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
// Gathers as coherent loads with a memory clobber, streaming stores with a
// memory clobber: ptxas may not sink a store below a later load that could
// alias it, so a batch of gathers stays issued back to back (memory-level
// parallelism) instead of being interleaved with the stores to save
// registers (which it does with .nc loads).
__device__ __forceinline__ uint2 ld_gather(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ uint4 ld_gather(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_stream(uint2* p, uint2 v) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream_u32(uint32_t* p, uint32_t v) { __stcs(p, v); }

// Row value -1 of a phased permutation: IEEE negation of both parts, done on
// the sign bits (bit-exact, NaN payloads kept; the oracle's -x).
__device__ __forceinline__ uint2 negate_if(uint2 v, uint32_t neg) {
  const uint32_t m = neg << 31;
  v.x ^= m;
  v.y ^= m;
  return v;
}
__device__ __forceinline__ uint4 negate_if(uint4 v, uint32_t neg) {  // two doubles
  const uint32_t m = neg << 31;
  v.y ^= m;
  v.w ^= m;
  return v;
}
__device__ __forceinline__ float2 negate_if(float2 v, uint32_t neg) {
  const uint32_t m = neg << 31;
  return make_float2(__uint_as_float(__float_as_uint(v.x) ^ m),
                     __uint_as_float(__float_as_uint(v.y) ^ m));
}
__device__ __forceinline__ double2 negate_if(double2 v, uint32_t neg) {
  const unsigned long long m = (unsigned long long)neg << 63;
  return make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ m),
                      __longlong_as_double(__double_as_longlong(v.y) ^ m));
}

// ------------------------------------------------------------------ per-lane
// One address per lane: walk the gates last -> first, x ^= tmask when all
// control bits of x are set.  APT independent walks interleave to fill the
// ALU pipe.
template <int CAP, int MODE, typename T, int APT>
__global__ void __launch_bounds__(256)
k_walk_per_lane(const __grid_constant__ GateList<CAP> g, uint64_t start, uint64_t count,
                uint32_t* __restrict__ perm_out, const T* __restrict__ k1,
                T* __restrict__ k2_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * APT;
  for (uint64_t r0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * APT; r0 < count;
       r0 += stride) {
    uint32_t x[APT], sg[APT];
#pragma unroll
    for (int a = 0; a < APT; ++a) {
      x[a] = (uint32_t)(start + r0 + a);
      sg[a] = 0u;
    }
    for (int k = (int)g.n - 1; k >= 0; --k) {
      const uint32_t w = g.w[k];
      const uint32_t kind = gate_kind(w), t = gate_t(w);
      const uint32_t tmask = 1u << t;
      if (kind == 6) {  // SWAP: exchange bits t and c0 (toggle both when they differ)
        const uint32_t c = gate_c0(w), both = tmask | (1u << c);
#pragma unroll
        for (int a = 0; a < APT; ++a) x[a] ^= (((x[a] >> t) ^ (x[a] >> c)) & 1u) ? both : 0u;
        continue;
      }
      const uint32_t nc = kind % 3;  // controls: NOT/Z 0, CNOT/CZ 1, CCNOT/CCZ 2
      const uint32_t cmask = (nc >= 1 ? (1u << gate_c0(w)) : 0u) | (nc == 2 ? (1u << gate_c1(w)) : 0u);
      if (kind >= 3) {  // phase: -1 on the rows with target and controls all 1
        const uint32_t pm = cmask | tmask;
#pragma unroll
        for (int a = 0; a < APT; ++a) sg[a] ^= (~x[a] & pm) == 0u ? 1u : 0u;
        continue;
      }
#pragma unroll
      for (int a = 0; a < APT; ++a)
        if ((~x[a] & cmask) == 0u) x[a] ^= tmask;
    }
#pragma unroll
    for (int a = 0; a < APT; ++a) {
      const uint64_t r = r0 + a;
      if (r < count) {
        if (MODE == 0) perm_out[r] = x[a];
        else k2_out[r] = negate_if(ld_gather(k1 + x[a]), sg[a]);
      }
    }
  }
}

// ------------------------------------------------------------ sigma tables
struct SigmaParams {
  uint8_t sigma[32];            // counter bit k -> output bit sigma[k] (bits 0..2 / 0..1 fixed)
  uint32_t chunk_log2;          // counters per CTA chunk
  uint32_t nbits;               // M
  unsigned long long* ticket;   // in-order chunk dispenser (zeroed), or null: grid-stride
};

// deposit tables: T[b][v] = OR over bits j of byte v of (1 << sigma[8b + j])
__device__ __forceinline__ void sigma_tables(const SigmaParams& sp, uint32_t (*T)[256]) {
  for (int x = threadIdx.x; x < 4 * 256; x += blockDim.x) {
    const int b = x >> 8, v = x & 255;
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (((v >> j) & 1) && 8 * b + j < (int)sp.nbits) r |= 1u << sp.sigma[8 * b + j];
    T[b][v] = r;
  }
}

__device__ __forceinline__ uint32_t sigma_apply(uint32_t (*T)[256], uint64_t c) {
  return T[0][c & 255] | T[1][(c >> 8) & 255] | T[2][(c >> 16) & 255] | T[3][(c >> 24) & 255];
}

// Next chunk for this CTA: in counter order from the ticket, else grid-stride.
__device__ __forceinline__ uint64_t next_chunk(const SigmaParams& sp, uint64_t cur,
                                               uint64_t* s_chunk, bool first) {
  if (sp.ticket) {
    __syncthreads();
    if (threadIdx.x == 0) *s_chunk = atomicAdd(sp.ticket, 1ull);
    __syncthreads();
    return *s_chunk;
  }
  return first ? (uint64_t)blockIdx.x : cur + gridDim.x;
}

// ---------------------------------------------------------------- bit-sliced
// A warp tile = 1024 counters: counter bits 0..4 are the lane, bits 5..9 the
// word bit l, bits >= 10 the tile.  Lane L, word bit l handles output
// out_base | Ltab[l] | sigma(L), where out_base = sigma(tile << 10) and
// Ltab[l] = sigma(l << 5).  Initial plane b of a thread: the lane bit that
// sigma maps to b (lanebit[b]), the standard 0xAAAAAAAA.. pattern if b is
// the image of an l-bit, else the (warp-uniform) bit b of out_base.
constexpr int kBsThreads = 256;
constexpr int kBsWarps = kBsThreads / 32;

// One block-swap stage: a[k] takes the low J-bit blocks of a[k] and a[k+J]
// shifted up, a[k+J] the high ones shifted down.  Stages 16 and 8 move whole
// bytes (two PRMT per pair); stages 4, 2, 1 a shift and a bit-select each.
template <int J, uint32_t MASK>
__device__ __forceinline__ void transpose_stage(uint32_t (&a)[32]) {
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if ((k & J) == 0) {
      const uint32_t x = a[k], y = a[k + J];
      if (J == 16) {
        a[k] = __byte_perm(x, y, 0x5410);
        a[k + J] = __byte_perm(x, y, 0x7632);
      } else if (J == 8) {
        a[k] = __byte_perm(x, y, 0x6240);
        a[k + J] = __byte_perm(x, y, 0x7351);
      } else {
        a[k] = (x & ~(MASK << J)) | ((y << J) & (MASK << J));
        a[k + J] = (y & ~MASK) | ((x >> J) & MASK);
      }
    }
  }
}

// In-register 32x32 bit transpose: on return bit b of a[l] = bit l of the
// input a[b].  Five block-swap stages (16, 8, 4, 2, 1).
__device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
  transpose_stage<16, 0x0000ffffu>(a);
  transpose_stage<8, 0x00ff00ffu>(a);
  transpose_stage<4, 0x0f0f0f0fu>(a);
  transpose_stage<2, 0x33333333u>(a);
  transpose_stage<1, 0x55555555u>(a);
}

struct BsShared {
  uint32_t S[34][kBsThreads];  // S[plane][thread] (private columns); 32 = ones, 33 = sign
  uint32_t tab[4][256];        // sigma deposit tables
  uint32_t patw[32];           // l-bit pattern of each output plane (0 if none)
  uint32_t ltab[32];           // sigma(l << 5)
  uint8_t lanebit[32];         // output plane b <- lane bit lanebit[b] (255: none)
  uint64_t chunk;
  uint2 gate[1];               // [n]: byte offsets of (target | c0 << 16, c1) planes
};

__host__ __device__ constexpr size_t bs_smem_bytes(uint32_t n) {
  return sizeof(BsShared) + (n > 0 ? n - 1 : 0) * sizeof(uint2);
}

template <int CAP>
__device__ __forceinline__ void bs_setup(const GateList<CAP>& g, const SigmaParams& sp,
                                         BsShared& sh) {
  sigma_tables(sp, sh.tab);
  const uint32_t pat[5] = {0xaaaaaaaau, 0xccccccccu, 0xf0f0f0f0u, 0xff00ff00u, 0xffff0000u};
  if (threadIdx.x < 32) {
    sh.patw[threadIdx.x] = 0;
    sh.lanebit[threadIdx.x] = 255;
  }
  sh.S[kOnesPlane][threadIdx.x] = 0xffffffffu;
  // gate list, last gate first (the walk order), as plane byte offsets
  for (uint32_t k = threadIdx.x; k < g.n; k += blockDim.x) {
    const uint32_t w = g.w[g.n - 1 - k];
    const uint32_t row = kBsThreads * 4u;
    sh.gate[k] = make_uint2((w & 0xffu) * row | (((w >> 8) & 0xffu) * row) << 16,
                            ((w >> 16) & 0xffu) * row | (w >> 24) << 16);
  }
  __syncthreads();
  if (threadIdx.x < 5 && 5 + threadIdx.x < sp.nbits) sh.patw[sp.sigma[5 + threadIdx.x]] = pat[threadIdx.x];
  if (threadIdx.x < 5 && threadIdx.x < sp.nbits) sh.lanebit[sp.sigma[threadIdx.x]] = (uint8_t)threadIdx.x;
  if (threadIdx.x < 32) {
    uint32_t o = 0;
    for (int j = 0; j < 5; ++j)
      if (((threadIdx.x >> j) & 1) && 5 + j < (int)sp.nbits) o |= 1u << sp.sigma[5 + j];
    sh.ltab[threadIdx.x] = o;
  }
  __syncthreads();
}

// Walk one warp tile; on return a[l] = perm(out_base | ltab[l] | sigma(lane))
// and bit l of sgn is 1 when that row's value is -1 (phase gates).
__device__ __forceinline__ void bs_walk_tile(uint32_t n, BsShared& sh, uint32_t out_base,
                                             uint32_t (&a)[32], uint32_t& sgn) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
#pragma unroll
  for (int b = 0; b < 32; ++b) {
    const uint32_t lb = sh.lanebit[b];
    const uint32_t lanew = (lb < 5) ? (((lane >> lb) & 1u) ? 0xffffffffu : 0u) : 0u;
    const uint32_t basew = ((out_base >> b) & 1u) ? 0xffffffffu : 0u;
    sh.S[b][tid] = lanew | sh.patw[b] | basew;
  }
  sh.S[kSignPlane][tid] = 0u;
  // walk last -> first (R1, R2): plane[t] ^= plane[c0] & plane[c1]; a SWAP
  // exchanges two planes; a phase gate adds plane[t] & plane[c0] & plane[c1]
  // to the sign plane (the op is warp-uniform)
  char* col = reinterpret_cast<char*>(&sh.S[0][tid]);
#pragma unroll 4
  for (uint32_t k = 0; k < n; ++k) {
    const uint2 gk = sh.gate[k];
    uint32_t* pt = reinterpret_cast<uint32_t*>(col + (gk.x & 0xffffu));
    uint32_t* p0 = reinterpret_cast<uint32_t*>(col + (gk.x >> 16));
    const uint32_t x1 = *reinterpret_cast<const uint32_t*>(col + (gk.y & 0xffffu));
    const uint32_t op = gk.y >> 16;
    if (op == kOpToggle) {
      *pt ^= *p0 & x1;
    } else if (op == kOpSwap) {
      const uint32_t d = *pt ^ *p0;
      *pt ^= d;
      *p0 ^= d;
    } else {
      sh.S[kSignPlane][tid] ^= *pt & *p0 & x1;
    }
  }
#pragma unroll
  for (int b = 0; b < 32; ++b) a[b] = sh.S[b][tid];
  sgn = sh.S[kSignPlane][tid];
  transpose32(a);
}

// MODE 0: perm_out[out - start] = perm(out) for out in [start, end), natural
// order (identity sigma), tiles [tile_begin, tile_end) grid-stride.  With
// signs_out (start % 32 == 0): bit r % 32 of signs_out[r / 32] = 1 when row
// start + r has value -1 (words of the range fully written, 0 past end).
template <int CAP>
__global__ void __launch_bounds__(kBsThreads, 2)
k_build_bitsliced(const __grid_constant__ GateList<CAP> g, const __grid_constant__ SigmaParams sp,
                  uint64_t start, uint64_t end, uint64_t tile_begin, uint64_t tile_end,
                  uint32_t* __restrict__ perm_out, uint32_t* __restrict__ signs_out) {
  extern __shared__ __align__(16) uint8_t bs_smem[];
  BsShared& sh = *reinterpret_cast<BsShared*>(bs_smem);
  bs_setup(g, sp, sh);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint64_t tile = tile_begin + (uint64_t)blockIdx.x * kBsWarps + warp; tile < tile_end;
       tile += (uint64_t)gridDim.x * kBsWarps) {
    const uint64_t base = tile << 10;
    uint32_t a[32], sgn;
    bs_walk_tile(g.n, sh, (uint32_t)base, a, sgn);
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const uint64_t addr = base + 32u * l + lane;
      if (addr >= start && addr < end) st_stream_u32(perm_out + (addr - start), a[l]);
    }
    if (signs_out) {  // row base + 32 l + lane: word l of the tile = ballot over lanes
      uint32_t mine = 0u;
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        const uint64_t addr = base + 32u * l + lane;
        const uint32_t b = __ballot_sync(0xffffffffu, addr < end && ((sgn >> l) & 1u));
        if ((uint32_t)l == lane) mine = b;
      }
      const uint64_t row = base + 32u * lane;  // first output of word `lane`
      if (row >= start && row < end) signs_out[(row - start) >> 5] = mine;
    }
  }
}

// Fused, natural order with an output range: k2_out[out - start] = k1[perm(out)].
template <int CAP, typename T>
__global__ void __launch_bounds__(kBsThreads, 2)
k_fused_bitsliced(const __grid_constant__ GateList<CAP> g, const __grid_constant__ SigmaParams sp,
                  uint64_t start, uint64_t end, uint64_t tile_begin, uint64_t tile_end,
                  const T* __restrict__ k1, T* __restrict__ k2_out) {
  extern __shared__ __align__(16) uint8_t bs_smem[];
  BsShared& sh = *reinterpret_cast<BsShared*>(bs_smem);
  bs_setup(g, sp, sh);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint64_t tile = tile_begin + (uint64_t)blockIdx.x * kBsWarps + warp; tile < tile_end;
       tile += (uint64_t)gridDim.x * kBsWarps) {
    const uint64_t base = tile << 10;
    uint32_t a[32], sgn;
    bs_walk_tile(g.n, sh, (uint32_t)base, a, sgn);
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
        if (addr >= start && addr < end)
          st_stream(k2_out + (addr - start), negate_if(v[l], (sgn >> (h + l)) & 1u));
      }
    }
  }
}

// Fused in sigma order over all 2^M outputs (M >= 10), chunks of
// 2^chunk_log2 counters taken from the ticket.
template <int CAP, typename T>
__global__ void __launch_bounds__(kBsThreads, 2)
k_fused_sigma(const __grid_constant__ GateList<CAP> g, const __grid_constant__ SigmaParams sp,
              uint64_t N, const T* __restrict__ k1, T* __restrict__ k2) {
  extern __shared__ __align__(16) uint8_t bs_smem[];
  BsShared& sh = *reinterpret_cast<BsShared*>(bs_smem);
  bs_setup(g, sp, sh);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t nchunks = N >> sp.chunk_log2;
  const uint32_t tiles_per_chunk = 1u << (sp.chunk_log2 - 10);
  for (uint64_t ch = next_chunk(sp, 0, &sh.chunk, true); ch < nchunks;
       ch = next_chunk(sp, ch, &sh.chunk, false)) {
    for (uint32_t tt = warp; tt < tiles_per_chunk; tt += kBsWarps) {
      const uint64_t c = (ch << sp.chunk_log2) + ((uint64_t)tt << 10);
      const uint32_t out_base = sigma_apply(sh.tab, c);
      const uint32_t lo = sh.tab[0][lane];
      uint32_t a[32], sgn;
      bs_walk_tile(g.n, sh, out_base, a, sgn);
      constexpr int B = sizeof(T) == 8 ? 32 : 16;  // gathers in flight per thread
#pragma unroll
      for (int h = 0; h < 32; h += B) {
        T v[B];
#pragma unroll
        for (int l = 0; l < B; ++l) v[l] = ld_gather(k1 + a[h + l]);
#pragma unroll
        for (int l = 0; l < B; ++l)
          st_stream(k2 + (out_base | sh.ltab[h + l] | lo), negate_if(v[l], (sgn >> (h + l)) & 1u));
      }
    }
  }
}

// ------------------------------------------------ input generated on the fly
// Appendix 1: k1(s) = q_M(b_M) ... q_1(b_1).  The M factors are
// grouped by bits of s into ng groups of gb bits (gb <= 11 for complex64,
// <= 8 for complex128; chosen on the host, kron_groups in qsim_api.cu):
// T_g[v] = product of q_j(bit) over the qubits of group g (j descending, the
// Kronecker order), and k1(s) = ((T_{ng-1} T_{ng-2}) ...) T_0, evaluated in
// the state precision, each complex product as re = fma(ar, br, -(ai*bi)),
// im = fma(ar, bi, ai*br) (error <= 2u per product; M - 1 products).
// The tables index bits of s in a chosen order (the layout, kron_layout in
// qsim_api.cu): table position k holds address bit pos[k] (identity unless
// permuted), so group g covers the bits pos[gb*g .. gb*g + gb - 1].  The
// product is the same set of factors in another grouping; every kernel of
// one call uses the same layout (identical bytes across kernels).
struct Qubits {
  double v[64][4];  // qubit j (1-based) at v[j-1]: re q(0), im q(0), re q(1), im q(1)
  uint32_t M;
  uint32_t gbits;   // bits per group
  uint32_t ngroups;
  uint8_t pos[64];  // table position -> address bit
  uint32_t permuted;
};

__device__ __forceinline__ float2 cmul_rn(float2 a, float2 b) {
  return make_float2(__fmaf_rn(a.x, b.x, -__fmul_rn(a.y, b.y)),
                     __fmaf_rn(a.x, b.y, __fmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
template <typename C> __device__ __forceinline__ C cmake(double re, double im);
template <> __device__ __forceinline__ float2 cmake<float2>(double re, double im) {
  return make_float2((float)re, (float)im);
}
template <> __device__ __forceinline__ double2 cmake<double2>(double re, double im) {
  return make_double2(re, im);
}

// Every thread of the CTA helps fill T[g << gbits | v] (call, then sync).
template <typename C>
__device__ __forceinline__ void kron_tables(const Qubits& q, C* T) {
  const int gb = (int)q.gbits;
  for (int x = threadIdx.x; x < ((int)q.ngroups << gb); x += blockDim.x) {
    const int g = x >> gb, v = x & ((1 << gb) - 1);
    C acc = cmake<C>(1.0, 0.0);
    bool first = true;
    for (int j = gb - 1; j >= 0; --j) {  // table position gb*g + j, descending
      const int k = gb * g + j;
      if (k >= (int)q.M) continue;
      const int b = q.pos[k], bit = (v >> j) & 1;
      const C f = cmake<C>(q.v[b][2 * bit], q.v[b][2 * bit + 1]);
      acc = first ? f : cmul_rn(acc, f);
      first = false;
    }
    T[x] = acc;
  }
}

template <typename C>
__device__ __forceinline__ C kron_element(const C* T, uint64_t s, const Qubits& q) {
  const uint32_t gb = q.gbits, ng = q.ngroups;
  if (q.permuted) {  // address bits to table positions
    uint64_t sp = 0;
    for (uint32_t k = 0; k < q.M; ++k) sp |= ((s >> q.pos[k]) & 1ull) << k;
    s = sp;
  }
  const uint64_t mask = (1ull << gb) - 1;
  C r = T[((ng - 1) << gb) | ((s >> (gb * (ng - 1))) & mask)];
  for (int g = (int)ng - 2; g >= 0; --g) r = cmul_rn(r, T[((uint32_t)g << gb) | ((s >> (gb * g)) & mask)]);
  return r;
}

__host__ __device__ constexpr size_t kron_table_bytes(uint32_t gbits, uint32_t ngroups,
                                                      size_t elem) {
  return ((size_t)ngroups << gbits) * elem;
}

// Fused with the map, natural order, output range [start, end):
// k2_out[out - start] = k1(perm(out)), k1 never stored (M <= 32).  Dynamic
// shared memory: BsShared (+ gates), then the product tables.
template <int CAP, typename C>
__global__ void __launch_bounds__(kBsThreads, 2)
k_fused_kron_bitsliced(const __grid_constant__ GateList<CAP> g,
                       const __grid_constant__ SigmaParams sp, const __grid_constant__ Qubits q,
                       uint64_t start, uint64_t end, uint64_t tile_begin, uint64_t tile_end,
                       C* __restrict__ k2_out) {
  extern __shared__ __align__(16) uint8_t bs_smem[];
  BsShared& sh = *reinterpret_cast<BsShared*>(bs_smem);
  C* T = reinterpret_cast<C*>(bs_smem + ((bs_smem_bytes(g.n) + 15) & ~(size_t)15));
  kron_tables<C>(q, T);
  bs_setup(g, sp, sh);  // ends with __syncthreads()
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint64_t tile = tile_begin + (uint64_t)blockIdx.x * kBsWarps + warp; tile < tile_end;
       tile += (uint64_t)gridDim.x * kBsWarps) {
    const uint64_t base = tile << 10;
    uint32_t a[32], sgn;
    bs_walk_tile(g.n, sh, (uint32_t)base, a, sgn);
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const uint64_t addr = base + 32u * l + lane;
      if (addr >= start && addr < end)
        k2_out[addr - start] =
            negate_if(kron_element<C>(T, a[l], q), (sgn >> l) & 1u);
    }
  }
}

// Any M <= 63 (64-bit addresses; output portions): one address per
// lane, the gates walked with 64-bit masks, the same product tables and
// order as the NVRTC kernels.  The fallback of qsim_run_fused_kron for
// M > 32 without NVRTC, and QSIM_WALK_PER_LANE.
template <int CAP, typename C>
__global__ void __launch_bounds__(256)
k_fused_kron_perlane64(const __grid_constant__ GateList<CAP> g, const __grid_constant__ Qubits q,
                       uint64_t start, uint64_t count, C* __restrict__ k2_out) {
  extern __shared__ __align__(16) uint8_t kt_smem[];
  C* T = reinterpret_cast<C*>(kt_smem);
  kron_tables<C>(q, T);
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += stride) {
    uint64_t x = start + r;
    uint32_t sg = 0u;
    for (int k = (int)g.n - 1; k >= 0; --k) {
      const uint32_t w = g.w[k], kind = gate_kind(w), t = gate_t(w);
      const uint64_t tm = 1ull << t;
      if (kind == 6) {
        const uint32_t c = gate_c0(w);
        if (((x >> t) ^ (x >> c)) & 1ull) x ^= tm | (1ull << c);
        continue;
      }
      const uint32_t nc = kind % 3;
      const uint64_t cm = (nc >= 1 ? 1ull << gate_c0(w) : 0ull) | (nc == 2 ? 1ull << gate_c1(w) : 0ull);
      if (kind >= 3) {
        sg ^= (~x & (cm | tm)) == 0ull ? 1u : 0u;
        continue;
      }
      if ((~x & cm) == 0ull) x ^= tm;
    }
    k2_out[r] = negate_if(kron_element<C>(T, x, q), sg);
  }
}

// --------------------------------------------------------------------- apply
// Natural order: k2[r] = k1[perm[r]]: perm streamed with 128-bit loads (4
// indices), the gathers issued back to back (8 in flight per thread).
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

// Phased form: k2[r] = sign[r] k1[perm[r]], bit r % 32 of signs[r / 32] = 1
// for -1 (qsim_apply_map_signed).  One thread per 4 entries.
template <typename T>
__global__ void __launch_bounds__(256)
k_apply_signed(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ signs,
               uint64_t count, const T* __restrict__ k1, T* __restrict__ k2) {
  const uint64_t ngroups = count >> 2;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups;
       gi += nthreads) {
    const uint4 p = ld_stream_u4(perm + 4 * gi);
    const uint32_t sw = signs[gi >> 3] >> (4u * (uint32_t)(gi & 7u));
    const T v0 = ld_gather(k1 + p.x), v1 = ld_gather(k1 + p.y);
    const T v2 = ld_gather(k1 + p.z), v3 = ld_gather(k1 + p.w);
    T* o = k2 + 4 * gi;
    st_stream(o + 0, negate_if(v0, sw & 1u));
    st_stream(o + 1, negate_if(v1, (sw >> 1) & 1u));
    st_stream(o + 2, negate_if(v2, (sw >> 2) & 1u));
    st_stream(o + 3, negate_if(v3, (sw >> 3) & 1u));
  }
  if (blockIdx.x == 0 && threadIdx.x < (count & 3u)) {
    const uint64_t r = (ngroups << 2) + threadIdx.x;
    k2[r] = negate_if(ld_gather(k1 + perm[r]), (signs[r >> 5] >> (r & 31u)) & 1u);
  }
}

// Sigma order (M >= 10): each warp takes U groups of 32 consecutive
// counters per iteration (perm: one 128-B line per group, k2: 256 B), chunks
// of 2^chunk_log2 counters from the ticket.
template <typename T, int U, int THREADS>
__global__ void __launch_bounds__(THREADS)
k_apply_sigma(const __grid_constant__ SigmaParams sp, const uint32_t* __restrict__ perm,
              uint64_t N, const T* __restrict__ k1, T* __restrict__ k2) {
  __shared__ uint32_t tab[4][256];
  __shared__ uint64_t s_chunk;
  sigma_tables(sp, tab);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t lo = tab[0][lane];  // sigma(lane)
  const uint64_t chunk = 1ull << sp.chunk_log2;
  const uint64_t nchunks = N >> sp.chunk_log2;
  for (uint64_t ch = next_chunk(sp, 0, &s_chunk, true); ch < nchunks;
       ch = next_chunk(sp, ch, &s_chunk, false)) {
    const uint64_t c0 = ch << sp.chunk_log2;
    for (uint64_t c = c0 + (uint64_t)warp * 32u * U; c < c0 + chunk;
         c += (uint64_t)nwarps * 32u * U) {
      uint32_t idx[U];
      uint32_t src[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        idx[u] = sigma_apply(tab, c + 32u * u) | lo;
        src[u] = __ldcs(perm + idx[u]);
      }
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_gather(k1 + src[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) st_stream(k2 + idx[u], v[u]);
    }
  }
}

}  // namespace qsim
