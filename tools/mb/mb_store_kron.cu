// mb_store_kron.cu -- microbenchmark (NOT the product path): the store pattern
// of the on-the-fly input kernel (qsim_jit_kron): 8-byte entries, lanes on
// output bits 0..4, a thread's 32 entries on the in-thread bits J, tiles of
// 1024 outputs over the other bits; 8 warps per CTA, 2 CTAs per SM.
// Variants: every warp stores its 32 entries in the same order, or in an
// order XOR-rotated by its warp / CTA index (the J streams then do not move
// in lockstep).  32 GiB buffer (2^32 complex64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_store_kron mb_store_kron.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 2) k_tile_j(uint2* out, uint64_t ntiles, int j0, int j1, int j2,
                                                   int j3, int j4, int rot) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const int J[5] = {j0, j1, j2, j3, j4};
  uint64_t offs[5];
  for (int k = 0; k < 5; ++k) offs[k] = 1ull << J[k];
  for (uint64_t tile = (uint64_t)blockIdx.x * 8u + warp; tile < ntiles; tile += (uint64_t)gridDim.x * 8u) {
    uint64_t base = tile << 5;
    for (int k = 0; k < 5; ++k) base = (base & ((1ull << J[k]) - 1)) | ((base >> J[k]) << (J[k] + 1));
    const uint32_t m = rot == 1 ? (warp * 4u) & 31u : rot == 2 ? (uint32_t)(tile & 31u) : 0u;
    uint64_t offm = 0;
    for (int k = 0; k < 5; ++k)
      if ((m >> k) & 1) offm |= offs[k];
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      uint64_t off = 0;
#pragma unroll
      for (int k = 0; k < 5; ++k)
        if ((l >> k) & 1) off |= offs[k];
      __stcs(out + base + (off ^ offm) + lane, make_uint2((uint32_t)l, 1u));
    }
  }
}

__global__ void k_seq(uint2* out, uint64_t n) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += nthr)
    __stcs(out + t, make_uint2(1u, 2u));
}

int main() {
  const uint64_t n = 1ull << 32, bytes = n * 8;
  uint2* out;
  if (cudaMalloc(&out, bytes) != cudaSuccess) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r && ms < best) best = ms;
    }
    printf("{\"case\": \"%s\", \"ms\": %.3f, \"GBps\": %.0f, \"err\": \"%s\"}\n", name, best,
           bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run("seq u64 grid=16xSM", [&] { k_seq<<<sms * 16, 256>>>(out, n); });
  const int Js[3][5] = {{7, 8, 13, 26, 29}, {5, 6, 7, 8, 9}, {9, 12, 16, 17, 23}};
  for (int t = 0; t < 3; ++t)
    for (int rot = 0; rot < 3; ++rot) {
      char nm[128];
      snprintf(nm, sizeof nm, "kron tiles J=%d.%d.%d.%d.%d rot=%s", Js[t][0], Js[t][1], Js[t][2], Js[t][3],
               Js[t][4], rot == 0 ? "none" : rot == 1 ? "warp" : "tile");
      run(nm, [&] { k_tile_j<<<sms * 8, 256>>>(out, n >> 10, Js[t][0], Js[t][1], Js[t][2], Js[t][3], Js[t][4], rot); });
    }
  cudaFree(out);
  return 0;
}
