// mb_window.cu -- microbenchmark (NOT the product path): the step's k1 read
// pattern in isolation.  Every 128-byte line of a 32 GiB buffer is read once,
// as its four 32-byte sectors, by different threads at different times: the
// lines are visited in a random order (a bijection), in windows of W lines;
// inside a window all lines' sector 0 are read, then sector 1, ... (so a
// line's sectors arrive W requests apart, well within L2 residency).  Loads
// plain or with the .L2::128B / .L2::256B prefetch-size qualifier.  Decides
// whether the L2 fetches a missing sector alone (four DRAM accesses per line)
// and whether the qualifier makes it fetch the line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_window mb_window.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x, int bits) {
  const uint64_t m = (1ull << bits) - 1;
  x = (x * 0x9e3779b97f4a7c15ull) & m;
  x ^= x >> (bits / 2);
  x = (x * 0xbf58476d1ce4e5b9ull) & m;
  x ^= x >> (bits / 3);
  x = (x * 0x94d049bb133111ebull) & m;
  return x;
}

template <int Q>
__device__ __forceinline__ uint4 ld32(const uint4* p) {  // first 16 B of a sector
  uint4 r;
  if (Q == 0)
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else if (Q == 1)
    asm volatile("ld.global.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else
    asm volatile("ld.global.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// request r (0 .. 4 * nlines): window w = r / (4W), visit t = (r / W) % 4,
// line = mix(w * W + r % W), sector (t + line) % 4 (the first-touched sector
// of a line is random).  PF: 0 none; 1 prefetch.global.L2 of the line by
// every request; 2 the same by sector-0 requests only; 3 cp.async.bulk
// prefetch of the 128-byte line by sector-0 requests
template <int Q, int PF>
__global__ void __launch_bounds__(256) win(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                           uint64_t nreq, int line_bits, int wbits) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nreq; r += stride) {
    const uint64_t w = r >> (wbits + 2), t = (r >> wbits) & 3, j = r & ((1ull << wbits) - 1);
    const uint64_t line = mix((w << wbits) | j, line_bits);
    const uint64_t c = (t + line) & 3;
    const uint4* lp = src + line * 8;
    if (PF == 1 || (PF == 2 && c == 0)) asm volatile("prefetch.global.L2 [%0];" ::"l"(lp));
    if (PF == 3 && c == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" ::"l"(lp) : "memory");
    const uint4 v = ld32<Q>(lp + c * 2);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x9e3779b9u) dst[0] = make_uint4(acc, 0, 0, 0);
}

// PF == 4: sector-0 requests copy the whole 128-byte line into shared memory
// with one TMA bulk copy (cp.async.bulk, mbarrier completion); every thread
// then still loads its own sector.  Is a bulk copy one line-sized L2 request?
__global__ void __launch_bounds__(256) win_tma(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                               uint64_t nreq, int line_bits, int wbits) {
  __shared__ __align__(128) uint4 slot[256][8];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t tid = threadIdx.x;
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_a), "r"(256u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0, phase = 0;
  for (uint64_t r0 = (uint64_t)blockIdx.x * blockDim.x; r0 < nreq; r0 += stride) {
    const uint64_t r = r0 + tid;
    const uint64_t w = r >> (wbits + 2), t = (r >> wbits) & 3, j = r & ((1ull << wbits) - 1);
    const uint64_t line = mix((w << wbits) | j, line_bits);
    const uint64_t c = (t + line) & 3;
    const uint4* lp = src + line * 8;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&slot[tid][0]);
    if (c == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 128;" ::"r"(bar_a) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                   ::"r"(sa), "l"(lp), "r"(bar_a) : "memory");
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_a) : "memory");
    }
    const uint4 v = ld32<0>(lp + c * 2);
    acc ^= v.x ^ v.w;
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 "@!P1 bra W_%=;\n}\n" ::"r"(bar_a), "r"(phase) : "memory");
    phase ^= 1u;
    acc ^= slot[tid][0].x;
  }
  if (acc == 0x9e3779b9u) dst[0] = make_uint4(acc, 0, 0, 0);
}

// PF == 5: the FIRST visit of each line (t == 0) is designated; the warp
// loads every designated line whole with cooperative instructions (four lanes
// per line, 16 bytes at each sector start: one instruction covers 8 lines),
// then every thread loads its own sector.  Emulates a traversal in which a
// line's first reader knows it is first.
__global__ void __launch_bounds__(256) win_coop(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                uint64_t nreq, int line_bits, int wbits) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t r0 = (uint64_t)blockIdx.x * blockDim.x; r0 < nreq; r0 += stride) {
    const uint64_t r = r0 + threadIdx.x;
    const uint64_t w = r >> (wbits + 2), t = (r >> wbits) & 3, j = r & ((1ull << wbits) - 1);
    const uint64_t line = mix((w << wbits) | j, line_bits);
    const uint64_t c = (t + line) & 3;
    const uint32_t mask = __ballot_sync(0xffffffffu, t == 0);
    const int nd = __popc(mask);
    for (int k = 0; k < nd; k += 8) {
      const int jd = k + (int)(lane >> 2);
      const int srcl = jd < nd ? (int)__fns(mask, 0, jd + 1) : 0;
      const uint64_t ln = __shfl_sync(0xffffffffu, line, srcl);
      if (jd < nd) {
        const uint4 v = ld32<0>(src + ln * 8 + (lane & 3u) * 2);
        acc ^= v.y;
      }
    }
    const uint4 v = ld32<0>(src + line * 8 + c * 2);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x9e3779b9u) dst[0] = make_uint4(acc, 0, 0, 0);
}

int main(int argc, char** argv) {
  const uint64_t BYTES = 32ull << 30, nlines = BYTES / 128, nreq = nlines * 4;
  int line_bits = 0;
  while ((1ull << line_bits) < nlines) ++line_bits;
  uint4 *src, *dst;
  if (cudaMalloc(&src, BYTES) != cudaSuccess || cudaMalloc(&dst, 64) != cudaSuccess) {
    printf("oom\n");
    return 1;
  }
  cudaMemset(src, 1, BYTES);
  {  // L2 fetch granularity: the default, then (argv[1]) the requested one
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity_default\": %zu}\n", g);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) {
    const cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity_set\": %s, \"now\": %zu, \"err\": \"%s\"}\n", argv[1], g,
           cudaGetErrorString(e));
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Case { int q, pf; const char* name; };
  const Case cases[] = {{0, 0, "-"}};
  [[maybe_unused]] const Case unused[] = {{1, 0, "ld.L2::128B"}, {0, 1, "prefetch.L2 every request"},
                        {0, 2, "prefetch.L2 by sector-0 requests"},
                        {0, 3, "cp.async.bulk.prefetch 128 B by sector-0 requests"}};
  const int bps = argc > 2 ? atoi(argv[2]) : 8;  // CTAs per SM (grid stride = time granularity)
  for (int wbits : {14, 16, 17, 19}) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      win_coop<<<sms * bps, 256>>>(src, dst, nreq, line_bits, wbits);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep && ms < best) best = ms;
    }
    printf("{\"window_lines\": %llu, \"ctas_per_sm\": %d, \"variant\": \"first visit: warp-cooperative whole-line load\", \"ms\": %.3f, \"line_GBps\": %.0f, \"err\": \"%s\"}\n",
           1ull << wbits, bps, best, BYTES / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  for (int wbits : {5, 10, 14}) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      win_tma<<<sms * bps, 256>>>(src, dst, nreq, line_bits, wbits);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep && ms < best) best = ms;
    }
    printf("{\"window_lines\": %llu, \"variant\": \"TMA bulk 128-B line copy by sector-0 requests\", \"ms\": %.3f, \"line_GBps\": %.0f, \"err\": \"%s\"}\n",
           1ull << wbits, best, BYTES / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  for (int wbits : {0, 4, 5, 10, 14, 19, 20}) {
    for (const Case& cs : cases) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (cs.q == 0 && cs.pf == 0) win<0, 0><<<sms * bps, 256>>>(src, dst, nreq, line_bits, wbits);
        if (cs.q == 1 && cs.pf == 0) win<1, 0><<<sms * bps, 256>>>(src, dst, nreq, line_bits, wbits);
        if (cs.pf == 1) win<0, 1><<<sms * bps, 256>>>(src, dst, nreq, line_bits, wbits);
        if (cs.pf == 2) win<0, 2><<<sms * bps, 256>>>(src, dst, nreq, line_bits, wbits);
        if (cs.pf == 3) win<0, 3><<<sms * bps, 256>>>(src, dst, nreq, line_bits, wbits);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
      }
      printf("{\"window_lines\": %llu, \"variant\": \"%s\", \"ms\": %.3f, \"line_GBps\": %.0f, \"err\": \"%s\"}\n",
             1ull << wbits, cs.name, best, BYTES / (best * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  }
  return 0;
}
