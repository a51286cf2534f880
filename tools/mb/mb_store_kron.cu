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

// 16-byte stores: a lane holds the two entries (o, o ^ 1) -- lanes on output
// bits 1..5, in-thread bits {0} + J[1..4]: 16 store instructions of 512 B
__global__ void __launch_bounds__(256, 2) k_tile_j16(uint4* out, uint64_t ntiles, int j1, int j2, int j3,
                                                     int j4) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const int J[5] = {0, j1, j2, j3, j4};
  for (uint64_t tile = (uint64_t)blockIdx.x * 8u + warp; tile < ntiles; tile += (uint64_t)gridDim.x * 8u) {
    uint64_t base = tile << 5;   // in units of entries, bits 1..5 = lane (entry pairs)
    for (int k = 1; k < 5; ++k) base = (base & ((1ull << J[k]) - 1)) | ((base >> J[k]) << (J[k] + 1));
    base = (base << 1);          // bit 0 is the pair
    // base now has lane bits at 6.. -- rebuild: lanes on bits 1..5
    uint64_t t = tile;
    uint64_t b2 = 0;
    int pos = 6, kk = 0;
    (void)kk;
    for (int bit = 6; bit < 40 && t; ++bit) {
      bool inJ = false;
      for (int k = 1; k < 5; ++k) inJ = inJ || (J[k] == bit);
      if (inJ) continue;
      b2 |= (t & 1ull) << bit;
      t >>= 1;
      (void)pos;
    }
    base = b2 | ((uint64_t)lane << 1);
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      uint64_t off = 0;
#pragma unroll
      for (int k = 1; k < 5; ++k)
        if ((l >> (k - 1)) & 1) off |= 1ull << J[k];
      __stcs(out + ((base + off) >> 1), make_uint4((uint32_t)l, 1u, 2u, 3u));
    }
  }
}

template <typename V>
__global__ void k_seqv(V* out, uint64_t n, V v) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += nthr) __stcs(out + t, v);
}

__global__ void k_seq(uint2* out, uint64_t n) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += nthr)
    __stcs(out + t, make_uint2(1u, 2u));
}

int main(int argc, char** argv) {
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
  if (argc > 1) {  // J sets given as a.b.c.d.e: the kernel's store pattern for each (rot none)
    for (int i = 1; i < argc; ++i) {
      int J[5];
      if (sscanf(argv[i], "%d.%d.%d.%d.%d", &J[0], &J[1], &J[2], &J[3], &J[4]) != 5) continue;
      char nm[128];
      snprintf(nm, sizeof nm, "kron tiles J=%s", argv[i]);
      run(nm, [&] { k_tile_j<<<sms * 8, 256>>>(out, n >> 10, J[0], J[1], J[2], J[3], J[4], 0); });
    }
    cudaFree(out);
    return 0;
  }
  run("seq u64 grid=16xSM", [&] { k_seq<<<sms * 16, 256>>>(out, n); });
  for (int g : {8, 16, 32}) {
    char nm[64];
    snprintf(nm, sizeof nm, "seq u64 grid=%dxSM", g);
    run(nm, [&] { k_seqv<uint2><<<sms * g, 256>>>(out, n, make_uint2(1u, 2u)); });
    snprintf(nm, sizeof nm, "seq u128 grid=%dxSM", g);
    run(nm, [&] { k_seqv<uint4><<<sms * g, 256>>>(reinterpret_cast<uint4*>(out), n / 2, make_uint4(1u, 2u, 3u, 4u)); });
  }
  run("kron tiles 16-B pairs J=0.7.13.26.29", [&] {
    k_tile_j16<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(out), n >> 10, 7, 13, 26, 29);
  });
  run("kron tiles 16-B pairs J=0.6.7.8.9", [&] {
    k_tile_j16<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(out), n >> 10, 6, 7, 8, 9);
  });
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
