// qsim_api.cu -- the C ABI declared in include/qsim.h: argument validation,
// gate packing into the kernel-parameter bank, launch configuration.
//
// Nothing here computes on the host beyond packing the gate list: every
// step of the path (walk, gather) runs in the kernels of qsim_kernels.cuh.
#include <cstdio>
#include <cstring>

#include "qsim.h"
#include "qsim_kernels.cuh"

namespace {

thread_local char g_err[512] = "";
thread_local int32_t g_launches = 0;

int cuda_fail(cudaError_t e, const char* what) {
  std::snprintf(g_err, sizeof g_err, "%s: %s (%s)", what, cudaGetErrorString(e),
                cudaGetErrorName(e));
  return QSIM_ECUDA;
}

#define QSIM_CHECK_LAUNCH(what)                          \
  do {                                                   \
    cudaError_t e_ = cudaGetLastError();                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);   \
    ++g_launches;                                        \
  } while (0)

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool overlap(const void* a, uint64_t abytes, const void* b, uint64_t bbytes) {
  if (abytes == 0 || bbytes == 0) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + bbytes && b0 < a0 + abytes;
}

int elem_bytes(int32_t dtype) { return dtype == QSIM_C64 ? 8 : dtype == QSIM_C128 ? 16 : 0; }

// Validate and pack the gate list (P:L43 semantics; readings R3-R5).
template <int CAP>
int pack_gates(const qsim_gate* gates, int32_t n, int32_t M, qsim::GateList<CAP>& out) {
  out.n = (uint32_t)n;
  for (int32_t k = 0; k < n; ++k) {
    const qsim_gate& g = gates[k];
    if (g.kind > 2) return QSIM_EINVAL;
    if (g.target >= M) return QSIM_EBIT;
    uint32_t c0 = 0, c1 = 0;
    if (g.kind >= 1) {
      if (g.c0 >= M || g.c0 == g.target) return QSIM_EBIT;
      c0 = g.c0;
    }
    if (g.kind == 2) {
      if (g.c1 >= M || g.c1 == g.target || g.c1 == g.c0) return QSIM_EBIT;
      c1 = g.c1;
    }
    out.w[k] = (uint32_t)g.kind | ((uint32_t)g.target << 8) | (c0 << 16) | (c1 << 24);
  }
  return QSIM_OK;
}

int check_gates_args(const qsim_gate* gates, int32_t n, int32_t M) {
  if (M < 1 || M > 32) return QSIM_ERANGE;
  if (n < 0 || n > QSIM_MAX_GATES) return QSIM_ECAP;
  if (n > 0 && gates == nullptr) return QSIM_EINVAL;
  return QSIM_OK;
}

int check_range(int32_t M, uint64_t start, uint64_t count) {
  const uint64_t N = 1ull << M;
  if (start > N || count > N - start) return QSIM_ERANGE;
  return QSIM_OK;
}

// Launch the walk (MODE 0: write perm, MODE 1: fused gather) with the
// gate list in a parameter bank sized for n.
template <int CAP, int MODE, typename T>
int launch_walk_cap(const qsim_gate* gates, int32_t n, int32_t M, uint64_t start, uint64_t count,
                    uint32_t* perm_out, const T* k1, T* k2_out, int32_t walk, cudaStream_t st) {
  qsim::GateList<CAP> gl;
  int rc = pack_gates<CAP>(gates, n, M, gl);
  if (rc != QSIM_OK) return rc;
  if (count == 0) return QSIM_OK;
  const int sms = sm_count();
  if (walk == QSIM_WALK_PER_LANE) {
    constexpr int APT = 4;
    const uint64_t threads = (count + APT - 1) / APT;
    uint64_t blocks = (threads + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8 * 16;
    if (blocks > cap) blocks = cap;
    qsim::k_walk_per_lane<CAP, MODE, T, APT><<<(unsigned)blocks, 256, 0, st>>>(
        gl, start, count, perm_out, k1, k2_out);
    QSIM_CHECK_LAUNCH("k_walk_per_lane");
  } else {
    const uint64_t tb = start >> 10, te = (start + count + 1023) >> 10;
    uint64_t blocks = (te - tb + qsim::kBsWarps - 1) / qsim::kBsWarps;
    const uint64_t cap = (uint64_t)sms * 6 * 32;
    if (blocks > cap) blocks = cap;
    qsim::k_walk_bitsliced<CAP, MODE, T><<<(unsigned)blocks, qsim::kBsThreads, 0, st>>>(
        gl, start, start + count, tb, te, perm_out, k1, k2_out);
    QSIM_CHECK_LAUNCH("k_walk_bitsliced");
  }
  return QSIM_OK;
}

template <int MODE, typename T>
int launch_walk(const qsim_gate* gates, int32_t n, int32_t M, uint64_t start, uint64_t count,
                uint32_t* perm_out, const T* k1, T* k2_out, int32_t walk, cudaStream_t st) {
  if (walk < 0 || walk > 2) return QSIM_EINVAL;
  if (n <= 64)
    return launch_walk_cap<64, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out, walk, st);
  if (n <= 256)
    return launch_walk_cap<256, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out, walk, st);
  if (n <= 1024)
    return launch_walk_cap<1024, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out, walk, st);
  return launch_walk_cap<qsim::kMaxGates, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out,
                                                   walk, st);
}

int build_impl(const qsim_gate* gates, int32_t n, int32_t M, uint64_t start, uint64_t count,
               uint32_t* perm_out, int32_t walk, cudaStream_t st) {
  int rc = check_gates_args(gates, n, M);
  if (rc) return rc;
  if ((rc = check_range(M, start, count))) return rc;
  if (perm_out == nullptr || !aligned16(perm_out)) return QSIM_EINVAL;
  return launch_walk<0, uint2>(gates, n, M, start, count, perm_out, nullptr, nullptr, walk, st);
}

int fused_impl(const qsim_gate* gates, int32_t n, int32_t M, int32_t dtype, uint64_t start,
               uint64_t count, const void* k1, void* k2, int32_t walk, cudaStream_t st) {
  int rc = check_gates_args(gates, n, M);
  if (rc) return rc;
  if ((rc = check_range(M, start, count))) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0) return QSIM_EINVAL;
  if (!k1 || !k2 || !aligned16(k1) || !aligned16(k2)) return QSIM_EINVAL;
  if (overlap(k1, (1ull << M) * e, k2, count * e)) return QSIM_EALIAS;
  if (dtype == QSIM_C64)
    return launch_walk<1, uint2>(gates, n, M, start, count, nullptr,
                                 static_cast<const uint2*>(k1), static_cast<uint2*>(k2), walk, st);
  return launch_walk<1, uint4>(gates, n, M, start, count, nullptr, static_cast<const uint4*>(k1),
                               static_cast<uint4*>(k2), walk, st);
}

int apply_impl(const uint32_t* perm, uint64_t count, int32_t M, int32_t dtype, const void* k1,
               void* k2, cudaStream_t st) {
  if (M < 1 || M > 32) return QSIM_ERANGE;
  if (count > (1ull << M)) return QSIM_ERANGE;
  const int e = elem_bytes(dtype);
  if (e == 0) return QSIM_EINVAL;
  if (!perm || !k1 || !k2 || !aligned16(perm) || !aligned16(k1) || !aligned16(k2))
    return QSIM_EINVAL;
  const uint64_t N = 1ull << M;
  if (overlap(k1, N * e, k2, count * e) || overlap(perm, count * 4, k2, count * e))
    return QSIM_EALIAS;
  if (count == 0) return QSIM_OK;
  const uint64_t groups = count / 4;
  uint64_t blocks = (groups + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * 8 * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  if (dtype == QSIM_C64)
    qsim::k_apply<uint2><<<(unsigned)blocks, 256, 0, st>>>(perm, count,
                                                          static_cast<const uint2*>(k1),
                                                          static_cast<uint2*>(k2));
  else
    qsim::k_apply<uint4><<<(unsigned)blocks, 256, 0, st>>>(perm, count,
                                                          static_cast<const uint4*>(k1),
                                                          static_cast<uint4*>(k2));
  QSIM_CHECK_LAUNCH("k_apply");
  return QSIM_OK;
}

}  // namespace

extern "C" {

int qsim_build_map(const qsim_gate* gates, int32_t n_gates, int32_t M, uint32_t* perm,
                   void* stream) {
  g_launches = 0;
  if (M < 1 || M > 32) return QSIM_ERANGE;
  return build_impl(gates, n_gates, M, 0, 1ull << M, perm, QSIM_WALK_AUTO,
                    static_cast<cudaStream_t>(stream));
}

int qsim_build_map_range(const qsim_gate* gates, int32_t n_gates, int32_t M, uint64_t start,
                         uint64_t count, uint32_t* perm_out, void* stream) {
  g_launches = 0;
  return build_impl(gates, n_gates, M, start, count, perm_out, QSIM_WALK_AUTO,
                    static_cast<cudaStream_t>(stream));
}

int qsim_build_map_ex(const qsim_gate* gates, int32_t n_gates, int32_t M, uint64_t start,
                      uint64_t count, uint32_t* perm_out, int32_t walk, void* stream) {
  g_launches = 0;
  return build_impl(gates, n_gates, M, start, count, perm_out, walk,
                    static_cast<cudaStream_t>(stream));
}

int qsim_apply_map(const uint32_t* perm, int32_t M, int32_t dtype, const void* k1, void* k2,
                   void* stream) {
  g_launches = 0;
  if (M < 1 || M > 32) return QSIM_ERANGE;
  return apply_impl(perm, 1ull << M, M, dtype, k1, k2, static_cast<cudaStream_t>(stream));
}

int qsim_apply_map_range(const uint32_t* perm_in, uint64_t count, int32_t M, int32_t dtype,
                         const void* k1, void* k2_out, void* stream) {
  g_launches = 0;
  return apply_impl(perm_in, count, M, dtype, k1, k2_out, static_cast<cudaStream_t>(stream));
}

int qsim_run_fused(const qsim_gate* gates, int32_t n_gates, int32_t M, int32_t dtype,
                   const void* k1, void* k2, void* stream) {
  g_launches = 0;
  if (M < 1 || M > 32) return QSIM_ERANGE;
  return fused_impl(gates, n_gates, M, dtype, 0, 1ull << M, k1, k2, QSIM_WALK_AUTO,
                    static_cast<cudaStream_t>(stream));
}

int qsim_run_fused_range(const qsim_gate* gates, int32_t n_gates, int32_t M, int32_t dtype,
                         uint64_t start, uint64_t count, const void* k1, void* k2_out,
                         void* stream) {
  g_launches = 0;
  return fused_impl(gates, n_gates, M, dtype, start, count, k1, k2_out, QSIM_WALK_AUTO,
                    static_cast<cudaStream_t>(stream));
}

int qsim_run_fused_ex(const qsim_gate* gates, int32_t n_gates, int32_t M, int32_t dtype,
                      uint64_t start, uint64_t count, const void* k1, void* k2_out, int32_t walk,
                      void* stream) {
  g_launches = 0;
  return fused_impl(gates, n_gates, M, dtype, start, count, k1, k2_out, walk,
                    static_cast<cudaStream_t>(stream));
}

int qsim_run_host(const qsim_gate* gates, int32_t n_gates, int32_t M, int32_t dtype, int32_t mode,
                  const void* k1_host, void* k2_host, void* k1_dev, void* k2_dev,
                  uint32_t* perm_dev, void* stream) {
  g_launches = 0;
  int rc = check_gates_args(gates, n_gates, M);
  if (rc) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0 || (mode != 0 && mode != 1)) return QSIM_EINVAL;
  if (!k1_host || !k2_host || !k1_dev || !k2_dev) return QSIM_EINVAL;
  if (mode == 0 && !perm_dev) return QSIM_EINVAL;
  const uint64_t N = 1ull << M, bytes = N * e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // validate the compute step before enqueuing anything
  if (!aligned16(k1_dev) || !aligned16(k2_dev) || (mode == 0 && !aligned16(perm_dev)))
    return QSIM_EINVAL;
  if (overlap(k1_dev, bytes, k2_dev, bytes) ||
      (mode == 0 && (overlap(perm_dev, N * 4, k2_dev, bytes) ||
                     overlap(perm_dev, N * 4, k1_dev, bytes))))
    return QSIM_EALIAS;
  {
    qsim::GateList<qsim::kMaxGates>* probe = new qsim::GateList<qsim::kMaxGates>;
    rc = pack_gates(gates, n_gates, M, *probe);
    delete probe;
    if (rc) return rc;
  }
  cudaError_t ce = cudaMemcpyAsync(k1_dev, k1_host, bytes, cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "H2D k1");
  int launches = 0;
  if (mode == 0) {
    rc = build_impl(gates, n_gates, M, 0, N, perm_dev, QSIM_WALK_AUTO, st);
    launches += g_launches;
    g_launches = 0;
    if (rc) return rc;
    rc = apply_impl(perm_dev, N, M, dtype, k1_dev, k2_dev, st);
  } else {
    rc = fused_impl(gates, n_gates, M, dtype, 0, N, k1_dev, k2_dev, QSIM_WALK_AUTO, st);
  }
  launches += g_launches;
  if (rc) return rc;
  ce = cudaMemcpyAsync(k2_host, k2_dev, bytes, cudaMemcpyDeviceToHost, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "D2H k2");
  ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return cuda_fail(ce, "qsim_run_host sync");
  g_launches = launches;
  return QSIM_OK;
}

int32_t qsim_last_launch_count(void) { return g_launches; }

const char* qsim_strerror(int32_t code) {
  switch (code) {
    case QSIM_OK: return "ok";
    case QSIM_EINVAL: return "invalid argument (null/misaligned pointer, bad dtype/mode/kind)";
    case QSIM_ERANGE: return "M outside [1, 32] or range outside [0, 2^M)";
    case QSIM_EBIT: return "gate bit out of range, target among controls, or duplicate control";
    case QSIM_ECAP: return "gate count outside [0, QSIM_MAX_GATES]";
    case QSIM_EALIAS: return "device buffers overlap";
    case QSIM_ECUDA: return "CUDA call failed (see qsim_last_error)";
    default: return "unknown qsim status";
  }
}

const char* qsim_last_error(void) { return g_err; }

int32_t qsim_abi_version(void) { return 1; }

}  // extern "C"
