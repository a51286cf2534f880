// mb_store.cu -- microbenchmark (NOT the product path): write-only bandwidth
// by store width and pattern, 16 GiB buffer.  Decides whether the build
// kernel (4-byte entries, one 128-byte line per warp store) is limited by its
// store granularity.  Patterns: "seq" = grid-stride over consecutive warp
// chunks; "tile" = the build kernel's layout (a warp writes 32 x 128 B =
// 4 KB per tile, tiles taken by warps in order).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_store mb_store.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int W>  // bytes per lane store: 4, 8, 16
__global__ void k_store(uint32_t* out, uint64_t nwords, uint32_t v) {
  const uint64_t per = W / 4;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * per < nwords; t += nthr) {
    if (W == 4) __stcs(out + t, v);
    if (W == 8) __stcs(reinterpret_cast<uint2*>(out) + t, make_uint2(v, v));
    if (W == 16) __stcs(reinterpret_cast<uint4*>(out) + t, make_uint4(v, v, v, v));
  }
}

// build-like: warp tile of 1024 words, 32 stores of 32 lanes x 4 B
__global__ void k_store_tile(uint32_t* out, uint64_t ntiles, uint32_t v) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint64_t tile = (uint64_t)blockIdx.x * 8u + warp; tile < ntiles; tile += (uint64_t)gridDim.x * 8u) {
    uint32_t* p = out + (tile << 10) + lane;
#pragma unroll
    for (int l = 0; l < 32; ++l) __stcs(p + 32 * l, v + l);
  }
}
// same tile, 16-B stores: lane holds 4 consecutive words, 8 stores of 512 B
__global__ void k_store_tile16(uint32_t* out, uint64_t ntiles, uint32_t v) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint64_t tile = (uint64_t)blockIdx.x * 8u + warp; tile < ntiles; tile += (uint64_t)gridDim.x * 8u) {
    uint4* p = reinterpret_cast<uint4*>(out + (tile << 10)) + lane;
#pragma unroll
    for (int l = 0; l < 8; ++l) __stcs(p + 32 * l, make_uint4(v + l, v, v, v));
  }
}

// build-like tile with in-thread bits J: lane = output bits 0..4, store l at
// the J-combination offset, tiles enumerate the other bits (zero-insertion)
__global__ void k_store_tile_j(uint32_t* out, uint64_t ntiles, uint32_t v, int j0, int j1, int j2,
                               int j3, int j4) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const int J[5] = {j0, j1, j2, j3, j4};
  for (uint64_t tile = (uint64_t)blockIdx.x * 8u + warp; tile < ntiles; tile += (uint64_t)gridDim.x * 8u) {
    uint64_t base = tile << 5;
    for (int k = 0; k < 5; ++k) base = (base & ((1ull << J[k]) - 1)) | ((base >> J[k]) << (J[k] + 1));
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      uint64_t off = 0;
#pragma unroll
      for (int k = 0; k < 5; ++k)
        if ((l >> k) & 1) off |= 1ull << J[k];
      __stcs(out + base + off + lane, v + l);
    }
  }
}

int main() {
  const uint64_t bytes = 16ull << 30, nwords = bytes / 4;
  uint32_t* out;
  cudaMalloc(&out, bytes);
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
  for (int k : {8, 16, 32}) {
    char n[64];
    snprintf(n, sizeof n, "seq u32 grid=%dxSM", k);
    run(n, [&] { k_store<4><<<sms * k, 256>>>(out, nwords, 1u); });
    snprintf(n, sizeof n, "seq u64 grid=%dxSM", k);
    run(n, [&] { k_store<8><<<sms * k, 256>>>(out, nwords, 1u); });
    snprintf(n, sizeof n, "seq u128 grid=%dxSM", k);
    run(n, [&] { k_store<16><<<sms * k, 256>>>(out, nwords, 1u); });
    snprintf(n, sizeof n, "tile u32 grid=%dxSM", k);
    run(n, [&] { k_store_tile<<<sms * k, 256>>>(out, nwords >> 10, 1u); });
    snprintf(n, sizeof n, "tile u128 grid=%dxSM", k);
    run(n, [&] { k_store_tile16<<<sms * k, 256>>>(out, nwords >> 10, 1u); });
  }
  const int Js[5][5] = {{5, 6, 7, 8, 9}, {7, 8, 13, 26, 29}, {11, 13, 22, 23, 24}, {8, 13, 15, 21, 29},
                        {5, 14, 21, 30, 31}};
  for (int t = 0; t < 5; ++t) {
    char n[96];
    snprintf(n, sizeof n, "tile u32 J=%d.%d.%d.%d.%d grid=8xSM", Js[t][0], Js[t][1], Js[t][2], Js[t][3], Js[t][4]);
    run(n, [&] { k_store_tile_j<<<sms * 8, 256>>>(out, nwords >> 10, 1u, Js[t][0], Js[t][1], Js[t][2], Js[t][3], Js[t][4]); });
  }
  cudaFree(out);
  return 0;
}
