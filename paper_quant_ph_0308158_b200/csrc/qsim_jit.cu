// qsim_jit.cu -- circuit-specialised walk kernels compiled at run time.
//
// The bit-sliced walk keeps 32 addresses per thread as 32 bit-plane words
// (qsim_kernels.cuh).  With a run-time gate list the planes must live in
// shared memory (dynamic indices); compiled for one circuit they live in
// registers and a step of the wiring diagram (toggle the target bit
// when all control bits are 1) is one LOP3 for 32 addresses:
//     p_t ^= p_c0 & p_c1        (CCNOT)      p_t ^= p_c (CNOT)
// and a NOT costs nothing: the generator tracks each plane's polarity and
// folds the inversion into the logic ops that read it (one final NOT per
// inverted plane).  Gates are emitted last -> first (readings R1, R2).
//
// NVRTC is loaded with dlopen (no link-time dependency); the compiled
// module is cached per circuit for the life of the process.  If NVRTC or
// the driver entry points are unavailable the caller falls back to the
// shared-memory interpreter kernel (still this library's own CUDA code).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "qsim_jit.h"

namespace qsim {
namespace {

// ---- NVRTC through dlopen -------------------------------------------------
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  void* h = nullptr;
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                          const char* const*) = nullptr;
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*log)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
  int major = 0, minor = 0;
  bool ok = false;
};

struct Driver {
  PFN_cuModuleLoadData_v2000 load = nullptr;
  PFN_cuModuleGetFunction_v2000 getfn = nullptr;
  PFN_cuLaunchKernel_v4000 launch = nullptr;
  PFN_cuFuncSetAttribute_v9000 setattr = nullptr;
  bool ok = false;
};

std::mutex g_mu;
Nvrtc g_nvrtc;
Driver g_drv;
bool g_init = false;
std::string g_status = "not initialised";

template <typename F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  return f != nullptr;
}

void init_locked() {
  if (g_init) return;
  g_init = true;
  if (const char* off = std::getenv("QSIM_NO_JIT")) {
    if (off[0] && off[0] != '0') {
      g_status = "disabled by QSIM_NO_JIT";
      return;
    }
  }
  // the toolkit's NVRTC first (an absolute path loads it even when torch has
  // already mapped its own, older libnvrtc.so.12 into the process)
  const char* cands[] = {std::getenv("QSIM_NVRTC"), "/usr/local/cuda/lib64/libnvrtc.so.12",
                         "libnvrtc.so.12", "libnvrtc.so"};
  for (const char* c : cands) {
    if (!c) continue;
    g_nvrtc.h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
    if (g_nvrtc.h) break;
  }
  if (!g_nvrtc.h) {
    g_status = "libnvrtc not found";
    return;
  }
  Nvrtc& n = g_nvrtc;
  n.ok = sym(n.h, "nvrtcCreateProgram", n.create) && sym(n.h, "nvrtcCompileProgram", n.compile) &&
         sym(n.h, "nvrtcGetCUBINSize", n.cubin_size) && sym(n.h, "nvrtcGetCUBIN", n.cubin) &&
         sym(n.h, "nvrtcGetProgramLogSize", n.log_size) &&
         sym(n.h, "nvrtcGetProgramLog", n.log) && sym(n.h, "nvrtcDestroyProgram", n.destroy);
  if (!n.ok) {
    g_status = "libnvrtc symbols missing";
    return;
  }
  nvrtcResult_t (*version)(int*, int*) = nullptr;
  if (sym(n.h, "nvrtcVersion", version)) version(&n.major, &n.minor);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  bool ok = true;
  ok = ok && cudaGetDriverEntryPoint("cuModuleLoadData", &p, cudaEnableDefault, &q) == cudaSuccess &&
       q == cudaDriverEntryPointSuccess;
  g_drv.load = reinterpret_cast<PFN_cuModuleLoadData_v2000>(p);
  ok = ok && cudaGetDriverEntryPoint("cuModuleGetFunction", &p, cudaEnableDefault, &q) ==
                 cudaSuccess && q == cudaDriverEntryPointSuccess;
  g_drv.getfn = reinterpret_cast<PFN_cuModuleGetFunction_v2000>(p);
  ok = ok && cudaGetDriverEntryPoint("cuLaunchKernel", &p, cudaEnableDefault, &q) == cudaSuccess &&
       q == cudaDriverEntryPointSuccess;
  g_drv.launch = reinterpret_cast<PFN_cuLaunchKernel_v4000>(p);
  ok = ok && cudaGetDriverEntryPoint("cuFuncSetAttribute", &p, cudaEnableDefault, &q) ==
                 cudaSuccess && q == cudaDriverEntryPointSuccess;
  g_drv.setattr = reinterpret_cast<PFN_cuFuncSetAttribute_v9000>(p);
  g_drv.ok = ok;
  g_status = ok ? "ready (nvrtc " + std::to_string(g_nvrtc.major) + "." + std::to_string(g_nvrtc.minor) + ")"
               : "driver entry points unavailable";
}

// ---- code generation --------------------------------------------------------
const char* kPrelude = R"(
typedef unsigned int u32;
typedef unsigned long long u64;
// Coherent loads with a memory clobber keep the 16 gathers of a batch
// issued back to back: ptxas may not sink a store below a later load that
// could alias it, so program order (16 loads, then 16 stores) survives
// (with .nc loads ptxas interleaves them with the stores to save registers,
// which throws away the memory-level parallelism).
__device__ __forceinline__ uint2 ldg(const uint2* p) {
  uint2 r; asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p)
                        : "memory");
  return r; }
__device__ __forceinline__ uint4 ldg(const uint4* p) {
  uint4 r; asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r; }
__device__ __forceinline__ void stcs(uint2* p, uint2 v) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory"); }
__device__ __forceinline__ void stcs(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory"); }
// row value -1 (phase gates): IEEE negation of both parts on the sign bits
__device__ __forceinline__ uint2 negate_if(uint2 v, u32 neg) {
  const u32 m = neg << 31; v.x ^= m; v.y ^= m; return v; }
__device__ __forceinline__ uint4 negate_if(uint4 v, u32 neg) {
  const u32 m = neg << 31; v.y ^= m; v.w ^= m; return v; }
__device__ __forceinline__ float2 negate_if(float2 v, u32 neg) {
  const u32 m = neg << 31;
  return make_float2(__uint_as_float(__float_as_uint(v.x) ^ m), __uint_as_float(__float_as_uint(v.y) ^ m)); }
__device__ __forceinline__ double2 negate_if(double2 v, u32 neg) {
  const u64 m = (u64)neg << 63;
  return make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ m),
                      __longlong_as_double(__double_as_longlong(v.y) ^ m)); }
// 32x32 bit transpose, one block-swap stage: afterwards bit b of a[l] = bit l
// of the input a[b].  Stages 16 and 8 move whole bytes: two PRMT per pair;
// stages 4, 2, 1: a shift and a bit-select (LOP3) per output word.
#define QSIM_TS(J, MASK, a)                                                     \
  _Pragma("unroll") for (int k = 0; k < 32; ++k)                                \
    if ((k & J) == 0) {                                                         \
      const u32 x_ = a[k], y_ = a[k + J];                                       \
      if (J == 16) { a[k] = __byte_perm(x_, y_, 0x5410); a[k + J] = __byte_perm(x_, y_, 0x7632); } \
      else if (J == 8) { a[k] = __byte_perm(x_, y_, 0x6240); a[k + J] = __byte_perm(x_, y_, 0x7351); } \
      else { a[k] = (x_ & ~((MASK) << J)) | ((y_ << J) & ((MASK) << J));        \
             a[k + J] = (y_ & ~(MASK)) | ((x_ >> J) & (MASK)); }                \
    }
)";

// Straight-line walk for one tile: planes p0..p31 in registers, gates last
// -> first (readings R1, R2).  A NOT costs nothing (the plane's polarity is
// tracked and folded into the ops that read it); a SWAP costs nothing (the
// two logical bits exchange variables); a phase step (Z / CZ / CCZ, R17) adds
// the AND of its planes to `sg` (bit l = row value -1), which the caller
// declares.  An epilogue moves logical bit b back into p<b>.
std::string walk_code(const uint32_t* w, int n, int M) {
  std::string s;
  const int np = M > 32 ? 64 : 32;  // planes (64-bit addresses for M > 32)
  int phys[64];
  bool inv[64];
  for (int b = 0; b < 64; ++b) {
    phys[b] = b;
    inv[b] = false;
  }
  char buf[200];
  auto ref = [&](uint32_t b) -> std::string {
    return std::string(inv[b] ? "~p" : "p") + std::to_string(phys[b]);
  };
  for (int k = n - 1; k >= 0; --k) {
    const uint32_t kind = w[k] & 0xffu, t = (w[k] >> 8) & 0xffu, c0 = (w[k] >> 16) & 0xffu,
                   c1 = w[k] >> 24;
    buf[0] = 0;
    switch (kind) {
      case 0: inv[t] = !inv[t]; break;
      case 1: std::snprintf(buf, sizeof buf, "  p%d ^= %s;\n", phys[t], ref(c0).c_str()); break;
      case 2:
        std::snprintf(buf, sizeof buf, "  p%d ^= %s & %s;\n", phys[t], ref(c0).c_str(),
                      ref(c1).c_str());
        break;
      case 3: std::snprintf(buf, sizeof buf, "  sg ^= %s;\n", ref(t).c_str()); break;
      case 4:
        std::snprintf(buf, sizeof buf, "  sg ^= %s & %s;\n", ref(t).c_str(), ref(c0).c_str());
        break;
      case 5:
        std::snprintf(buf, sizeof buf, "  sg ^= %s & %s & %s;\n", ref(t).c_str(), ref(c0).c_str(),
                      ref(c1).c_str());
        break;
      case 6:
        std::swap(phys[t], phys[c0]);
        std::swap(inv[t], inv[c0]);
        break;
      default: break;
    }
    s += buf;
  }
  bool moved = false;
  for (int b = 0; b < np; ++b) moved = moved || phys[b] != b;
  if (moved) {  // parallel copy back to p<b>
    s += "  {\n";
    for (int b = 0; b < np; ++b) {
      std::snprintf(buf, sizeof buf, "    const u32 q%d = %s;\n", b, ref(b).c_str());
      s += buf;
    }
    for (int b = 0; b < np; ++b) {
      std::snprintf(buf, sizeof buf, "    p%d = q%d;\n", b, b);
      s += buf;
    }
    s += "  }\n";
  } else {
    for (int b = 0; b < np; ++b)
      if (inv[b]) {
        std::snprintf(buf, sizeof buf, "  p%d = ~p%d;\n", b, b);
        s += buf;
      }
  }
  (void)M;
  return s;
}

// In-thread output bits (qsim_api.cu thread_bits): a warp tile is 1024
// outputs = lanes on output bits 0..4 x the 32 bit positions of each plane on
// output bits J[0..4]; tiles enumerate the other bits, 2^(L-10) tiles per
// aligned block of 2^L outputs.  Stores stay 128 / 256-byte warp runs.
std::string thread_defs(const uint8_t* J, int L) {
  char buf[320];
  // streaming stores (write-back / .cg / .wt measured the same for the
  // on-the-fly input: profiles/r02_kron_store_policy.txt)
  const std::string st = "#define QSIM_ST(p, v) __stcs(p, v)\n";
  std::snprintf(buf, sizeof buf,
                "#define QSIM_L %d\n"
                "#define QSIM_OFF(l) (((l) & 1 ? 1ull << %d : 0ull) | ((l) & 2 ? 1ull << %d : 0ull) | "
                "((l) & 4 ? 1ull << %d : 0ull) | ((l) & 8 ? 1ull << %d : 0ull) | "
                "((l) & 16 ? 1ull << %d : 0ull))\n",
                L, J[0], J[1], J[2], J[3], J[4]);
  return st + buf;
}

// base = the tile's first output (lane and J bits clear), the initial planes
// (address bits of the 32 x 32 outputs), the tile's block test
std::string thread_planes(int M, const uint8_t* J, int np) {
  std::string s = "    u64 base = tile << 5;\n";
  char buf[200];
  for (int k = 0; k < 5; ++k) {  // insert a zero at each in-thread bit, ascending
    std::snprintf(buf, sizeof buf, "    base = (base & 0x%llxull) | ((base >> %d) << %d);\n",
                  (unsigned long long)((1ull << J[k]) - 1), J[k], J[k] + 1);
    s += buf;
  }
  const char* pat[5] = {"0xaaaaaaaau", "0xccccccccu", "0xf0f0f0f0u", "0xff00ff00u", "0xffff0000u"};
  for (int b = 0; b < np; ++b) {
    int jk = -1;
    for (int k = 0; k < 5; ++k)
      if (J[k] == b) jk = k;
    if (b >= M)
      std::snprintf(buf, sizeof buf, "    u32 p%d = 0u;\n", b);
    else if (b < 5)
      std::snprintf(buf, sizeof buf, "    u32 p%d = ((lane >> %d) & 1u) ? 0xffffffffu : 0u;\n", b, b);
    else if (jk >= 0)
      std::snprintf(buf, sizeof buf, "    u32 p%d = %s;\n", b, pat[jk]);
    else
      std::snprintf(buf, sizeof buf, "    u32 p%d = ((base >> %d) & 1ull) ? 0xffffffffu : 0u;\n", b, b);
    s += buf;
  }
  s += "    const u64 blk = base >> QSIM_L;\n"
       "    const bool full = (blk << QSIM_L) >= start && ((blk + 1ull) << QSIM_L) <= end;\n";
  return s;
}

// the 32 outputs of a thread: `value` defines rv for entry l; stores hoisted
// out of the range test for whole blocks
std::string thread_stores(const char* ptr, const char* value, const char* ind) {
  const std::string i(ind);
  std::string e;
  e += i + "auto* const kq = " + ptr + " + (base + lane - start);\n";
  e += i + "if (full) {\n";
  e += i + "  _Pragma(\"unroll\") for (int l = 0; l < 32; ++l) {\n";
  e += i + "    " + value + "\n";
  e += i + "    QSIM_ST(kq + QSIM_OFF(l), rv);\n";
  e += i + "  }\n";
  e += i + "} else {\n";
  e += i + "  _Pragma(\"unroll\") for (int l = 0; l < 32; ++l) {\n";
  e += i + "    const u64 addr = base + lane + QSIM_OFF(l);\n";
  e += i + "    if (addr >= start && addr < end) {\n";
  e += i + "      " + value + "\n";
  e += i + "      QSIM_ST(kq + QSIM_OFF(l), rv);\n";
  e += i + "    }\n";
  e += i + "  }\n";
  e += i + "}\n";
  return e;
}

// transpose stages over the array `a`
std::string transpose_code(const char* a, const char* ind) {
  char buf[320];
  std::snprintf(buf, sizeof buf,
                "%sQSIM_TS(16, 0x0000ffffu, %s) QSIM_TS(8, 0x00ff00ffu, %s) QSIM_TS(4, 0x0f0f0f0fu, %s)\n"
                "%sQSIM_TS(2, 0x33333333u, %s) QSIM_TS(1, 0x55555555u, %s)\n",
                ind, a, a, a, ind, a, a);
  return buf;
}

// The map: perm_out[out - start] = source of output out, M <= 32.
// Fast path (V != 0): when every address bit outside V is constant across a
// thread's 32 outputs and every bit in V is an affine function of the
// thread's output bits J (checked per warp tile), the 32 sources follow from
// one source and 5 difference columns, one XOR each; otherwise the 32x32
// transpose.
std::string build_source(const uint32_t* w, int n, int M, const uint8_t* J, int L, uint64_t V) {
  std::string s = kPrelude;
  s += thread_defs(J, L);
  s += R"(
extern "C" __global__ void __launch_bounds__(256)
qsim_jit_build(u64 start, u64 end, u64 tb, u64 te, u32* __restrict__ perm_out) {
  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (u64 tile = tb + (u64)blockIdx.x * 8u + warp; tile < te; tile += (u64)gridDim.x * 8u) {
)";
  char buf[512];
  s += thread_planes(M, J, 32);
  s += "    u32 sg = 0u;\n";
  s += walk_code(w, n, M);
  if (V != 0) {
    // affine fast path: every plane outside V constant in the thread, every
    // plane in V an affine function of the thread's 5 output bits (checked
    // with a bit-parallel XOR subset transform); then the 32 sources are
    // s0 ^ (XOR of the columns of the set bits of l), taken in Gray-code
    // order: one XOR per entry, no transpose
    s += "    u32 un = 0u, s0 = 0u, c0 = 0u, c1 = 0u, c2 = 0u, c3 = 0u, c4 = 0u;\n";
    for (int b = 0; b < M; ++b) {
      if ((V >> b) & 1ull) {
        std::snprintf(buf, sizeof buf,
                      "    { const u32 d = p%d ^ (0u - (p%d & 1u)); u32 h = d & 0x00010116u;\n"
                      "      h ^= (h << 1) & 0xaaaaaaaau; h ^= (h << 2) & 0xccccccccu; "
                      "h ^= (h << 4) & 0xf0f0f0f0u;\n"
                      "      h ^= (h << 8) & 0xff00ff00u; h ^= (h << 16) & 0xffff0000u; un |= h ^ d;\n",
                      b, b);
        s += buf;
        std::snprintf(buf, sizeof buf,
                      "      s0 |= (p%d & 1u) << %d; c0 |= ((d >> 1) & 1u) << %d; "
                      "c1 |= ((d >> 2) & 1u) << %d;\n"
                      "      c2 |= ((d >> 4) & 1u) << %d; c3 |= ((d >> 8) & 1u) << %d; "
                      "c4 |= ((d >> 16) & 1u) << %d; }\n",
                      b, b, b, b, b, b, b);
        s += buf;
      } else {
        std::snprintf(buf, sizeof buf, "    un |= p%d ^ (u32)((int)p%d >> 31); s0 |= p%d & 0x%xu;\n",
                      b, b, b, 1u << b);
        s += buf;
      }
    }
    s += "    if (__all_sync(0xffffffffu, un == 0u)) {\n";
    s += "      u32* const kq = perm_out + (base + lane - start);\n";
    for (int pass = 0; pass < 2; ++pass) {
      s += pass == 0 ? "      if (full) {\n" : "      } else {\n";
      s += "        u32 sv = s0;\n";
      for (int t = 0; t < 32; ++t) {
        const int l = t ^ (t >> 1);
        if (t) {
          const int k = __builtin_ctz((unsigned)t);
          std::snprintf(buf, sizeof buf, "        sv ^= c%d;\n", k);
          s += buf;
        }
        if (pass == 0)
          std::snprintf(buf, sizeof buf, "        __stcs(kq + QSIM_OFF(%d), sv);\n", l);
        else
          std::snprintf(buf, sizeof buf,
                        "        { const u64 addr = base + lane + QSIM_OFF(%d); "
                        "if (addr >= start && addr < end) __stcs(kq + QSIM_OFF(%d), sv); }\n",
                        l, l);
        s += buf;
      }
    }
    s += "      }\n      continue;\n    }\n";
  }
  s += "    u32 a[32] = {";
  for (int b = 0; b < 32; ++b) {
    std::snprintf(buf, sizeof buf, "p%d%s", b, b < 31 ? ", " : "};\n");
    s += buf;
  }
  s += transpose_code("a", "    ");
  s += thread_stores("perm_out", "const u32 rv = a[l];", "    ");
  s += "  }\n}\n";
  return s;
}

// Sigma-ordered fused walk + gather (qsim_kernels.cuh k_fused_sigma, with the
// circuit compiled in).  If perm_out is non-null the kernel also stores the
// map (one-pass materialised map + gather); from_perm: the planned apply, the
// sources read from a stored map instead of walked.
//
// Counter c -> output sigma(c): counter bits 0..4 are the lanes, 5..9 the 32
// entries a thread holds (bit positions of its planes), 10.. the warp tile,
// the CTA's 8 warps and the chunk.  Only sigma[0..9] shape the generated
// code (which output bits are lane / word bits); the rest of sigma is a
// kernel parameter (the tile offset `ob` comes from 4 shared-memory tables
// built from it), so qsim_plan_tune can try orders of the high counter bits
// without recompiling.
// ident: sigma is the identity over all M positions (natural order; the
// kernel then skips the order tables -- the runtime tail is ignored)
std::string fused_source(const uint32_t* w, int n, int M, const uint8_t* sigma, int elem,
                         bool from_perm, int warps = 8, bool ident = false) {
  std::string s = kPrelude;
  char buf[256];
  std::snprintf(buf, sizeof buf, "#define QSIM_T %s\n#define QSIM_M %d\n#define QSIM_B %d\n#define QSIM_W %du\n"
                "#define QSIM_IDENT %d\n#define QSIM_TICKET_AHEAD %d\n",
                elem == 8 ? "uint2" : "uint4", M, elem == 8 ? 32 : 16, warps, ident ? 1 : 0,
                from_perm ? 0 : 1);  // ticket ahead: gather -1.5 %, apply +1.5 % (r02_ticket_ahead_ab.json)
  s += buf;
  s += from_perm ? "#define QSIM_KNAME qsim_jit_apply\n" : "#define QSIM_KNAME qsim_jit_fused\n";
  s += R"(
struct Sigma { unsigned char s[32]; };
extern "C" __global__ void __launch_bounds__(32 * QSIM_W)
QSIM_KNAME(u64 N, u32 chunk_log2, u64* ticket, const QSIM_T* __restrict__ k1,
           QSIM_T* __restrict__ k2, u32* __restrict__ perm_out, const Sigma sig) {
  __shared__ u64 s_chunk[2];
#if QSIM_IDENT   // natural order: output = counter, no tables
  (void)sig;
#else
  __shared__ u32 tab[4][256];
  for (int x = threadIdx.x; x < 1024; x += blockDim.x) {
    const int b = x >> 8, v = x & 255;
    u32 r = 0;
    for (int j = 0; j < 8; ++j)
      if (((v >> j) & 1) && 8 * b + j < QSIM_M) r |= 1u << sig.s[8 * b + j];
    tab[b][v] = r;
  }
  __syncthreads();
#endif
  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const u64 nchunks = N >> chunk_log2;
  const u32 tiles = 1u << (chunk_log2 - 10);
  // chunks in counter order: from a device ticket (dynamic), or without a
  // workspace round-robin by CTA (static; the front still moves in order)
#if QSIM_TICKET_AHEAD
  // the ticket of the next chunk is taken while this one is worked on (one
  // barrier per chunk; the atomic's round trip is not waited for by the CTA)
  if (ticket && threadIdx.x == 0) s_chunk[0] = atomicAdd(ticket, 1ull);
#endif
  for (u64 it = 0;; ++it) {
    u64 ch;
    if (ticket) {
#if QSIM_TICKET_AHEAD
      __syncthreads();  // chunk it-1 done by every warp, slot it&1 written
      ch = s_chunk[it & 1];
      if (threadIdx.x == 0 && ch < nchunks) s_chunk[(it + 1) & 1] = atomicAdd(ticket, 1ull);
#else
      __syncthreads();
      if (threadIdx.x == 0) s_chunk[0] = atomicAdd(ticket, 1ull);
      __syncthreads();
      ch = s_chunk[0];
#endif
    } else {
      ch = (u64)blockIdx.x + it * gridDim.x;
    }
    if (ch >= nchunks) break;
    for (u32 tt = warp; tt < tiles; tt += QSIM_W) {
      const u64 c = (ch << chunk_log2) + ((u64)tt << 10);
#if QSIM_IDENT
      const u32 ob = (u32)c;
#else
      const u32 ob = tab[0][c & 255] | tab[1][(c >> 8) & 255] | tab[2][(c >> 16) & 255] |
                     tab[3][(c >> 24) & 255];
#endif
)";
  if (!from_perm) {
    // plane initialisation: output bit b comes from counter bit inv[b]: a
    // lane bit (< 5), a word bit (5..9, compile-time pattern) or a tile bit
    // (ob); then the walk and the transpose: a[l] = source of entry l
    const char* pat[5] = {"0xaaaaaaaau", "0xccccccccu", "0xf0f0f0f0u", "0xff00ff00u", "0xffff0000u"};
    uint8_t inv[32];
    for (int b = 0; b < 32; ++b) inv[b] = 255;
    for (int k = 0; k < M; ++k) inv[sigma[k]] = (uint8_t)k;
    for (int b = 0; b < 32; ++b) {
      const int c = b < M ? inv[b] : 255;
      if (c < 5)
        std::snprintf(buf, sizeof buf, "      u32 p%d = ((lane >> %d) & 1u) ? 0xffffffffu : 0u;\n", b, c);
      else if (c < 10)
        std::snprintf(buf, sizeof buf, "      u32 p%d = %s;\n", b, pat[c - 5]);
      else if (c < 32)
        std::snprintf(buf, sizeof buf, "      u32 p%d = ((ob >> %d) & 1u) ? 0xffffffffu : 0u;\n", b, b);
      else
        std::snprintf(buf, sizeof buf, "      u32 p%d = 0u;\n", b);
      s += buf;
    }
    s += "      u32 sg = 0u;\n";
    s += walk_code(w, n, M);
    s += "      u32 a[32] = {";
    for (int b = 0; b < 32; ++b) {
      std::snprintf(buf, sizeof buf, "p%d%s", b, b < 31 ? ", " : "};\n");
      s += buf;
    }
    s += "      QSIM_TS(16, 0x0000ffffu, a) QSIM_TS(8, 0x00ff00ffu, a) QSIM_TS(4, 0x0f0f0f0fu, a)\n";
    s += "      QSIM_TS(2, 0x33333333u, a) QSIM_TS(1, 0x55555555u, a)\n";
  }
  // output offsets of the 32 word bits: sigma(l << 5), compile-time
  s += "      const u32 lt[32] = {";
  for (int l = 0; l < 32; ++l) {
    uint32_t o = 0u;
    for (int j = 0; j < 5 && 5 + j < M; ++j)
      if ((l >> j) & 1) o ^= 1u << sigma[5 + j];
    std::snprintf(buf, sizeof buf, "%uu%s", o, l < 31 ? ", " : "};\n");
    s += buf;
  }
  s += R"(
#if QSIM_IDENT
      const u32 lo = lane;
#else
      const u32 lo = tab[0][lane];   // output bits of the lane: sigma(lane)
#endif
)";
  if (from_perm)  // the apply: sources read from the materialised map (32-B runs)
    s += R"(
      u32 a[32];
      const u32 sg = 0u;
      _Pragma("unroll") for (int l = 0; l < 32; ++l) a[l] = __ldcs(perm_out + (ob ^ lt[l] ^ lo));
)";
  else
    s += R"(
      if (perm_out) {
        _Pragma("unroll") for (int l = 0; l < 32; ++l) __stcs(perm_out + (ob ^ lt[l] ^ lo), a[l]);
      }
)";
  s += R"(
      _Pragma("unroll") for (int h = 0; h < 32; h += QSIM_B) {
        QSIM_T v[QSIM_B];
        _Pragma("unroll") for (int l = 0; l < QSIM_B; ++l) v[l] = ldg(k1 + a[h + l]);
        _Pragma("unroll") for (int l = 0; l < QSIM_B; ++l)
          stcs(k2 + (ob ^ lt[h + l] ^ lo), negate_if(v[l], (sg >> (h + l)) & 1u));
      }
    }
  }
}
)";
  return s;
}

// Fused walk with the input generated on the fly (Appendix 1):
// k2_out[out - start] = k1(perm(out)) from tables of qubit products, ng
// groups of gb table positions (same arithmetic and order as
// qsim_kernels.cuh kron_tables / kron_element: each complex product
// re = fma(ar, br, -(ai*bi)), im = fma(ar, bi, ai*br)); table position k holds
// address bit pos[k] of the source.  M > 32 (64-bit addresses; SURVEY 8f
// NEXT(2), "continuous portions"): 64 planes.
//
// Traversal (the layout, chosen on the host by kron_layout): a warp tile is
// 1024 outputs = lanes on output bits 0..4 x the 32 bit positions of each
// plane on output bits J[0..4]; tiles enumerate the other bits, 2^(L-10)
// tiles per aligned block of 2^L outputs.  Stores stay 256-byte warp runs.
// Fast path (nv > 0): when every source bit at table positions >= nv is
// constant across a thread's 32 entries (checked per warp tile; the host
// picked J so that it nearly always is), the product of groups ng-1..1 is
// formed once per thread and each entry takes one lookup and one complex
// product: cmul(C, T_0[x]) -- the same operations, in the same order, as the
// general path, so both give identical bytes.
std::string kron_source(const uint32_t* w, int n, int M, int elem, int gb, int ng,
                        const uint8_t* pos, const uint8_t* J, int L, int nv) {
  std::string s = kPrelude;
  char buf[640];
  const bool f32 = elem == 8, wide = M > 32;
  s += f32 ? "typedef float2 C; typedef float R;\n" : "typedef double2 C; typedef double R;\n";
  std::snprintf(buf, sizeof buf, "#define QSIM_M %d\n#define QSIM_GB %d\n#define QSIM_NG %d\n", M, gb,
                ng);
  s += buf;
  s += thread_defs(J, L);
  s += f32 ? R"(
__device__ __forceinline__ C cmul(C a, C b) {
  return make_float2(__fmaf_rn(a.x, b.x, -__fmul_rn(a.y, b.y)),
                     __fmaf_rn(a.x, b.y, __fmul_rn(a.y, b.x))); }
)" : R"(
__device__ __forceinline__ C cmul(C a, C b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x))); }
)";
  s += R"(
struct Qubits { double v[64][4]; u32 M, gbits, ngroups; unsigned char pos[64]; u32 permuted; };
extern "C" __global__ void __launch_bounds__(256, 1)
qsim_jit_kron(u64 start, u64 end, u64 tb, u64 te, Qubits q, C* __restrict__ k2) {
  extern __shared__ __align__(16) unsigned char kt_smem[];
  C* T = reinterpret_cast<C*>(kt_smem);   // [QSIM_NG << QSIM_GB]
  for (int x = threadIdx.x; x < (QSIM_NG << QSIM_GB); x += blockDim.x) {
    const int g = x >> QSIM_GB, v = x & ((1 << QSIM_GB) - 1);
    C acc; bool first = true;
    for (int j = QSIM_GB - 1; j >= 0; --j) {
      const int k = QSIM_GB * g + j;
      if (k >= QSIM_M) continue;
      const int b = q.pos[k], bit = (v >> j) & 1;
      C f; f.x = (R)q.v[b][2 * bit]; f.y = (R)q.v[b][2 * bit + 1];
      acc = first ? f : cmul(acc, f);
      first = false;
    }
    if (first) { acc.x = (R)1; acc.y = (R)0; }
    T[x] = acc;
  }
  __syncthreads();
  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (u64 tile = tb + (u64)blockIdx.x * 8u + warp; tile < te; tile += (u64)gridDim.x * 8u) {
)";
  const int np = wide ? 64 : 32;
  s += thread_planes(M, J, np);
  s += "    u32 sg = 0u;\n";
  s += walk_code(w, n, M);
  auto P = [&](int k) { return std::string("p") + std::to_string(pos[k]); };

  if (nv > 0 && ng >= 2) {
    s += "    u32 un = 0u;\n";
    for (int k = nv; k < M; ++k) {
      std::snprintf(buf, sizeof buf, "    un |= %s ^ (u32)((int)%s >> 31);\n", P(k).c_str(), P(k).c_str());
      s += buf;
    }
    s += "    if (__all_sync(0xffffffffu, un == 0u)) {\n";
    for (int g = 0; g < ng; ++g) {
      std::snprintf(buf, sizeof buf, "      u32 i%d = 0u;\n", g);
      s += buf;
      for (int j = 0; j < gb; ++j) {
        const int k = gb * g + j;
        if (k >= M || k < nv) continue;
        std::snprintf(buf, sizeof buf, "      i%d |= %s & 0x%xu;\n", g, P(k).c_str(), 1u << j);
        s += buf;
      }
    }
    std::snprintf(buf, sizeof buf, "      C cc = T[%d | i%d];\n", (ng - 1) << gb, ng - 1);
    s += buf;
    for (int g = ng - 2; g >= 1; --g) {
      std::snprintf(buf, sizeof buf, "      cc = cmul(cc, T[%d | i%d]);\n", g << gb, g);
      s += buf;
    }
    s += "      u32 a[32] = {";
    for (int k = 0; k < 32; ++k) {
      s += k < nv ? P(k) : std::string("0u");
      s += k < 31 ? ", " : "};\n";
    }
    s += "      QSIM_TS(16, 0x0000ffffu, a) QSIM_TS(8, 0x00ff00ffu, a) QSIM_TS(4, 0x0f0f0f0fu, a)\n";
    s += "      QSIM_TS(2, 0x33333333u, a) QSIM_TS(1, 0x55555555u, a)\n";
    s += thread_stores("k2", "const C rv = negate_if(cmul(cc, T[a[l] | i0]), (sg >> l) & 1u);", "      ");
    s += "      continue;\n    }\n";
  }
  for (int h = 0; h < (wide ? 2 : 1); ++h) {
    std::snprintf(buf, sizeof buf, "    u32 a%d[32] = {", h);
    s += buf;
    for (int b = 0; b < 32; ++b) {
      const int k = 32 * h + b;
      s += k < M ? P(k) : std::string("0u");
      s += b < 31 ? ", " : "};\n";
    }
    std::snprintf(buf, sizeof buf,
                  "    QSIM_TS(16, 0x0000ffffu, a%d) QSIM_TS(8, 0x00ff00ffu, a%d) "
                  "QSIM_TS(4, 0x0f0f0f0fu, a%d)\n    QSIM_TS(2, 0x33333333u, a%d) "
                  "QSIM_TS(1, 0x55555555u, a%d)\n", h, h, h, h, h);
    s += buf;
  }
  s += wide ? "#define QSIM_SRC(l) (((u64)a1[l] << 32) | a0[l])\n"
            : "#define QSIM_SRC(l) ((u64)a0[l])\n";
  s += "    const u64 gm = (1ull << QSIM_GB) - 1;\n";
  std::string gen = "const u64 sv = QSIM_SRC(l);";
  std::snprintf(buf, sizeof buf, " C r = T[%d | ((sv >> %d) & gm)];", (ng - 1) << gb, gb * (ng - 1));
  gen += buf;
  for (int g = ng - 2; g >= 0; --g) {
    std::snprintf(buf, sizeof buf, " r = cmul(r, T[%d | ((sv >> %d) & gm)]);", g << gb, gb * g);
    gen += buf;
  }
  gen += " const C rv = negate_if(r, (sg >> l) & 1u);";
  s += thread_stores("k2", gen.c_str(), "    ");
  s += "  }\n}\n";
  return s;
}

// Circuits that keep locality (every target / SWAP bit below T): each aligned
// tile of 2^T outputs reads exactly the same tile of k1 (the walk never
// changes bits >= T).  One CTA per SM streams tiles: a TMA bulk copy
// (cp.async.bulk, mbarrier completion) brings tile i+1 of k1 into shared
// memory while the 8 warps walk tile i (planes in registers), read their
// sources from shared memory and write k2 (and perm) with fully coalesced
// 256-byte warp stores -- the gather of the north star "staged in shared
// memory where the circuit keeps locality".
std::string local_source(const uint32_t* w, int n, int M, int elem, int T) {
  std::string s = kPrelude;
  char buf[256];
  std::snprintf(buf, sizeof buf, "#define QSIM_M %d\n#define QSIM_LT %d\ntypedef %s E;\n", M, T,
                elem == 8 ? "uint2" : "uint4");
  s += buf;
  s += R"(
__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
extern "C" __global__ void __launch_bounds__(256, 1)
qsim_jit_local(u64 ntiles, const E* __restrict__ k1, E* __restrict__ k2, u32* __restrict__ perm_out) {
  extern __shared__ __align__(128) unsigned char lsm[];      // 2 stages x 2^T entries
  __shared__ __align__(8) u64 bar[2];
  const u32 tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const u32 TILE = 1u << QSIM_LT, BYTES = (u32)sizeof(E) << QSIM_LT;
  E* stage0 = reinterpret_cast<E*>(lsm);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&bar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&bar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](u64 t, u32 st) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&bar[st])), "r"(BYTES) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_addr(stage0 + st * TILE)), "l"(k1 + (t << QSIM_LT)), "r"(BYTES),
                    "r"(smem_addr(&bar[st])) : "memory");
  };
  if (tid == 0 && (u64)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  u32 i = 0;
  for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    const u32 st = i & 1u;
    if (tid == 0 && t + gridDim.x < ntiles) issue(t + gridDim.x, st ^ 1u);
    {
      const u32 bp = smem_addr(&bar[st]), par = (i >> 1) & 1u;
      asm volatile("{\n.reg .pred P1;\nLW_%=:\n"
                   "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                   "@!P1 bra LW_%=;\n}\n" :: "r"(bp), "r"(par) : "memory");
    }
    const E* sv = stage0 + st * TILE;
    for (u32 wt = warp; wt < (TILE >> 10); wt += 8u) {
      const u64 base = (t << QSIM_LT) | ((u64)wt << 10);
)";
  const char* pat[5] = {"0xaaaaaaaau", "0xccccccccu", "0xf0f0f0f0u", "0xff00ff00u", "0xffff0000u"};
  for (int b = 0; b < 32; ++b) {
    if (b >= M)
      std::snprintf(buf, sizeof buf, "      u32 p%d = 0u;\n", b);
    else if (b < 5)
      std::snprintf(buf, sizeof buf, "      u32 p%d = ((lane >> %d) & 1u) ? 0xffffffffu : 0u;\n", b, b);
    else if (b < 10)
      std::snprintf(buf, sizeof buf, "      u32 p%d = %s;\n", b, pat[b - 5]);
    else
      std::snprintf(buf, sizeof buf, "      u32 p%d = ((base >> %d) & 1ull) ? 0xffffffffu : 0u;\n", b, b);
    s += buf;
  }
  s += "      u32 sg = 0u;\n";
  s += walk_code(w, n, M);
  s += "      u32 a[32] = {";
  for (int b = 0; b < 32; ++b) {
    std::snprintf(buf, sizeof buf, "p%d%s", b, b < 31 ? ", " : "};\n");
    s += buf;
  }
  s += "      QSIM_TS(16, 0x0000ffffu, a) QSIM_TS(8, 0x00ff00ffu, a) QSIM_TS(4, 0x0f0f0f0fu, a)\n";
  s += "      QSIM_TS(2, 0x33333333u, a) QSIM_TS(1, 0x55555555u, a)\n";
  s += R"(
      if (perm_out) {
        _Pragma("unroll") for (int l = 0; l < 32; ++l) __stcs(perm_out + base + 32u * l + lane, a[l]);
      }
      _Pragma("unroll") for (int l = 0; l < 32; ++l)
        stcs(k2 + base + 32u * l + lane, negate_if(sv[a[l] & (TILE - 1u)], (sg >> l) & 1u));
    }
    __syncthreads();   // the stage is refilled two tiles later
  }
}
)";
  return s;
}

struct Entry {
  std::vector<uint32_t> words;
  int M;
  CUfunction fn;
  double compile_ms;
};
std::unordered_map<uint64_t, std::vector<Entry>> g_cache;
// compiles that failed, with their error: not retried on every call
std::unordered_map<uint64_t, std::vector<std::pair<std::vector<uint32_t>, std::string>>> g_failed;
double g_last_compile_ms = 0.0;

uint64_t fnv(const uint32_t* w, int n, uint64_t salt) {
  uint64_t h = 1469598103934665603ull ^ salt;
  for (int k = 0; k < n; ++k) {
    h ^= w[k];
    h *= 1099511628211ull;
  }
  return h;
}

bool compile_cubin_locked(const std::string& src, std::vector<char>& cubin, std::string& err) {
  Nvrtc& nv = g_nvrtc;
  nvrtcProgram_t prog = nullptr;
  if (nv.create(&prog, src.c_str(), "qsim_jit.cu", 0, nullptr, nullptr) != 0) {
    err = "nvrtcCreateProgram failed";
    return false;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-default-device", "--std=c++17",
                        "-lineinfo"};
  const int rc = nv.compile(prog, 4, opts);
  if (rc != 0) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    err = "nvrtc compile failed: " + log.substr(0, 400);
    nv.destroy(&prog);
    return false;
  }
  size_t cs = 0;
  nv.cubin_size(prog, &cs);
  cubin.resize(cs);
  nv.cubin(prog, cubin.data());
  nv.destroy(&prog);
  if (const char* dir = std::getenv("QSIM_JIT_DUMP")) {  // debugging aid
    const std::string base = std::string(dir) + "/qsim_jit_" + std::to_string(src.size());
    if (FILE* f = std::fopen((base + ".cu").c_str(), "w")) {
      std::fwrite(src.data(), 1, src.size(), f);
      std::fclose(f);
    }
    if (FILE* f = std::fopen((base + ".cubin").c_str(), "wb")) {
      std::fwrite(cubin.data(), 1, cubin.size(), f);
      std::fclose(f);
    }
  }
  return true;
}

CUfunction compile_locked(const std::string& src, const char* name, std::string& err) {
  std::vector<char> cubin;
  if (!compile_cubin_locked(src, cubin, err)) return nullptr;
  CUmodule mod = nullptr;
  if (g_drv.load(&mod, cubin.data()) != CUDA_SUCCESS) {
    err = "cuModuleLoadData failed";
    return nullptr;
  }
  CUfunction fn = nullptr;
  if (g_drv.getfn(&fn, mod, name) != CUDA_SUCCESS) {
    err = "cuModuleGetFunction failed";
    return nullptr;
  }
  // the walk kernels use <= 5 KB of static shared memory: give the rest of
  // the unified array to L1 (the gather's reuse cache)
  g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 3);
  return fn;
}

}  // namespace

bool jit_available() {
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  return g_nvrtc.ok && g_drv.ok;
}

const char* jit_status() {
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  return g_status.c_str();
}

double jit_last_compile_ms() { return g_last_compile_ms; }

// Find or compile the kernel for (kind, words, M, extra); extra is folded
// into the key words (sigma, element size).
CUfunction get_kernel_locked(uint64_t kind, const std::vector<uint32_t>& keyw, int M,
                             const std::string& src, const char* name, std::string& err) {
  const uint64_t key = fnv(keyw.data(), (int)keyw.size(), kind);
  for (const Entry& e : g_cache[key])
    if (e.M == M && e.words == keyw) return e.fn;
  std::vector<uint32_t> fkey(keyw);
  fkey.push_back((uint32_t)M);
  for (const auto& f : g_failed[key])
    if (f.first == fkey) {
      err = f.second;
      return nullptr;
    }
  const auto t0 = std::chrono::steady_clock::now();
  CUfunction fn = compile_locked(src, name, err);
  if (!fn) {
    g_failed[key].push_back({fkey, err});
    return nullptr;
  }
  g_last_compile_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  g_cache[key].push_back(Entry{keyw, M, fn, g_last_compile_ms});
  return fn;
}

int jit_check_compile(const uint32_t* words, int n, int M, const uint8_t* J, int L, uint64_t V,
                      std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  if (!g_nvrtc.ok) {
    err = g_status;
    return -1;
  }
  std::vector<char> cubin;
  return compile_cubin_locked(build_source(words, n, M, J, L, V), cubin, err) ? 0 : -1;
}

// words: per-lane gate format (kind | t << 8 | c0 << 16 | c1 << 24).
int jit_build(const uint32_t* words, int n, int M, const uint8_t* J, int L, uint64_t V,
              uint64_t start, uint64_t count, uint32_t* perm_out, int sms, cudaStream_t st,
              std::string& err) {
  CUfunction fn = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    if (!(g_nvrtc.ok && g_drv.ok)) {
      err = g_status;
      return -1;
    }
    std::vector<uint32_t> keyw(words, words + n);
    for (int k = 0; k < 5; ++k) keyw.push_back(J[k]);
    keyw.push_back((uint32_t)L);
    keyw.push_back((uint32_t)V);
    keyw.push_back((uint32_t)(V >> 32));
    const uint64_t kind = 0x6275696c64ull;
    const uint64_t key = fnv(keyw.data(), (int)keyw.size(), kind);
    for (const Entry& e : g_cache[key])
      if (e.M == M && e.words == keyw) fn = e.fn;
    if (!fn) {
      fn = get_kernel_locked(kind, keyw, M, build_source(words, n, M, J, L, V), "qsim_jit_build",
                             err);
      if (!fn) return -1;
    }
  }
  if (count == 0) return 0;
  // whole blocks of 2^L outputs (the tiles of a block interleave its outputs)
  uint64_t end = start + count;
  uint64_t tb = (start >> L) << (L - 10), te = ((end + (1ull << L) - 1) >> L) << (L - 10);
  uint64_t blocks = (te - tb + 7) / 8;
  const uint64_t cap = (uint64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  void* args[] = {&start, &end, &tb, &te, &perm_out};
  if (g_drv.launch(fn, (unsigned)blocks, 1, 1, 256, 1, 1, 0, (CUstream)st, args, nullptr) !=
      CUDA_SUCCESS) {
    err = "cuLaunchKernel failed";
    return -1;
  }
  return 0;
}

namespace {
// the kernel parameter carrying the whole traversal order (see fused_source)
struct SigmaArg {
  unsigned char s[32];
};

// one chunk ticket reset + launch of a gather kernel (fused / apply)
int launch_gather(CUfunction fn, int M, const uint8_t* sigma, uint32_t chunk_log2, const void* k1,
                  void* k2, uint32_t* perm, void* ticket, int blocks, int warps, cudaStream_t st,
                  std::string& err) {
  uint64_t N = 1ull << M;
  uint32_t cl = chunk_log2;
  SigmaArg sg;
  std::memcpy(sg.s, sigma, 32);
  void* args[] = {&N, &cl, &ticket, const_cast<void**>(&k1), &k2, &perm, &sg};
  if (ticket && cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), st) != cudaSuccess) {
    err = "ticket reset failed";
    return -1;
  }
  if (g_drv.launch(fn, (unsigned)blocks, 1, 1, 32u * (unsigned)warps, 1, 1, 0, (CUstream)st, args, nullptr) !=
      CUDA_SUCCESS) {
    err = "cuLaunchKernel failed";
    return -1;
  }
  return 0;
}

// cache key of a gather kernel: what shapes its code (sigma[0..9], the dtype
// and, for the fused walk, the gates)
bool sigma_ident(const uint8_t* sigma, int M) {
  for (int k = 0; k < M && k < 32; ++k)
    if (sigma[k] != k) return false;
  return true;
}

std::vector<uint32_t> gather_key(const uint32_t* words, int n, const uint8_t* sigma, int elem, int warps,
                                 int M) {
  std::vector<uint32_t> keyw(words, words + n);
  keyw.push_back(sigma_ident(sigma, M) ? 1u : 0u);
  for (int k = 0; k < 10; ++k) keyw.push_back(sigma[k]);
  keyw.push_back((uint32_t)elem);
  keyw.push_back((uint32_t)warps);
  return keyw;
}
}  // namespace

int jit_fused(const uint32_t* words, int n, int M, const uint8_t* sigma, uint32_t chunk_log2,
              int elem, const void* k1, void* k2, uint32_t* perm_out, void* ticket, int blocks,
              int warps, cudaStream_t st, std::string& err) {
  CUfunction fn = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    if (!(g_nvrtc.ok && g_drv.ok)) {
      err = g_status;
      return -1;
    }
    const std::vector<uint32_t> keyw = gather_key(words, n, sigma, elem, warps, M);
    const uint64_t kind = 0x66757365ull;
    const uint64_t key = fnv(keyw.data(), (int)keyw.size(), kind);
    for (const Entry& e : g_cache[key])  // the source is only generated on a cache miss
      if (e.M == M && e.words == keyw) fn = e.fn;
    if (!fn)
      fn = get_kernel_locked(kind, keyw, M, fused_source(words, n, M, sigma, elem, false, warps, sigma_ident(sigma, M)),
                             "qsim_jit_fused", err);
    if (!fn) return -1;
  }
  return launch_gather(fn, M, sigma, chunk_log2, k1, k2, perm_out, ticket, blocks, warps, st, err);
}

// NVRTC programs are independent, so several compile at once (the driver
// calls that load the modules stay under the lock).
int jit_fused_prepare(const uint32_t* words, int n, int M, const uint8_t* sigmas, int count, int elem,
                      int warps, int threads, bool apply) {
  // apply: the planned-apply kernels of those orders (jit_apply's key / source)
  const uint64_t kind = apply ? 0x6170706c79ull : 0x66757365ull;
  if (apply) {
    words = nullptr;
    n = 0;
  }
  std::vector<std::vector<uint32_t>> keys;
  std::vector<std::string> srcs;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    if (!(g_nvrtc.ok && g_drv.ok)) return -1;
    for (int i = 0; i < count; ++i) {
      const uint8_t* sg = sigmas + 32 * i;
      std::vector<uint32_t> keyw = gather_key(words, n, sg, elem, warps, M);
      const uint64_t key = fnv(keyw.data(), (int)keyw.size(), kind);
      bool have = false;
      for (const Entry& e : g_cache[key]) have = have || (e.M == M && e.words == keyw);
      for (const auto& k : keys) have = have || k == keyw;
      if (have) continue;
      keys.push_back(keyw);
      srcs.push_back(fused_source(words, n, M, sg, elem, apply, warps, sigma_ident(sg, M)));
    }
  }
  const size_t m = keys.size();
  std::vector<std::vector<char>> cubins(m);
  std::vector<std::string> errs(m);
  std::vector<char> ok(m, 0);
  std::atomic<size_t> next{0};
  auto work = [&]() {
    for (size_t i; (i = next.fetch_add(1)) < m;) ok[i] = compile_cubin_locked(srcs[i], cubins[i], errs[i]);
  };
  const int nt = (int)std::min<size_t>(m, (size_t)std::max(1, threads));
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) {
    try {
      pool.emplace_back(work);
    } catch (...) {  // no more threads: the ones running (and this one) finish the list
      break;
    }
  }
  work();
  for (auto& t : pool) t.join();
  int done = 0;
  std::lock_guard<std::mutex> lk(g_mu);
  for (size_t i = 0; i < m; ++i) {
    if (!ok[i]) continue;  // jit_fused compiles it again and reports the error
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    if (g_drv.load(&mod, cubins[i].data()) != CUDA_SUCCESS ||
        g_drv.getfn(&fn, mod, apply ? "qsim_jit_apply" : "qsim_jit_fused") != CUDA_SUCCESS)
      continue;
    g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 3);
    const uint64_t key = fnv(keys[i].data(), (int)keys[i].size(), kind);
    g_cache[key].push_back(Entry{keys[i], M, fn, 0.0});
    ++done;
  }
  return done;
}

int jit_kron(const uint32_t* words, int n, int M, const void* qubits_struct, size_t qbytes,
             int elem, int gbits, int ngroups, const uint8_t* pos, const uint8_t* J, int L, int nv,
             uint64_t start, uint64_t count, void* k2_out, int sms, cudaStream_t st,
             std::string& err) {
  const int smem = (ngroups << gbits) * (elem == 8 ? 8 : 16);
  CUfunction fn = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    if (!(g_nvrtc.ok && g_drv.ok)) {
      err = g_status;
      return -1;
    }
    std::vector<uint32_t> keyw(words, words + n);
    keyw.push_back((uint32_t)elem);
    keyw.push_back((uint32_t)gbits);
    keyw.push_back((uint32_t)ngroups);
    for (int k = 0; k < M; ++k) keyw.push_back(pos[k]);
    for (int k = 0; k < 5; ++k) keyw.push_back(J[k]);
    keyw.push_back((uint32_t)L);
    keyw.push_back((uint32_t)nv);
    const uint64_t kind = 0x6b726f6eull;
    const uint64_t key = fnv(keyw.data(), (int)keyw.size(), kind);
    for (const Entry& e : g_cache[key])
      if (e.M == M && e.words == keyw) fn = e.fn;
    if (!fn) {
      fn = get_kernel_locked(kind, keyw, M, kron_source(words, n, M, elem, gbits, ngroups, pos, J, L, nv),
                             "qsim_jit_kron", err);
      if (!fn) return -1;
      // write-only: shared memory for the tables of several resident CTAs
      // (the gather kernels' 3 % carveout would allow one)
      g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 50);
      if (g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem) != CUDA_SUCCESS) {
        err = "cuFuncSetAttribute(max dynamic smem) failed";
        return -1;
      }
    }
  }
  if (count == 0) return 0;
  // whole blocks of 2^L outputs (the tiles of a block interleave its outputs)
  uint64_t end = start + count;
  uint64_t tb = (start >> L) << (L - 10), te = ((end + (1ull << L) - 1) >> L) << (L - 10);
  uint64_t blocks = (te - tb + 7) / 8;
  const uint64_t cap = (uint64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  (void)qbytes;
  void* args[] = {&start, &end, &tb, &te, const_cast<void*>(qubits_struct), &k2_out};
  if (g_drv.launch(fn, (unsigned)blocks, 1, 1, 256, 1, 1, (unsigned)smem, (CUstream)st, args,
                   nullptr) != CUDA_SUCCESS) {
    err = "cuLaunchKernel failed";
    return -1;
  }
  return 0;
}

int jit_check_compile_kron(const uint32_t* words, int n, int M, int elem, int gbits, int ngroups,
                           const uint8_t* pos, const uint8_t* J, int L, int nv, std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  if (!g_nvrtc.ok) {
    err = g_status;
    return -1;
  }
  std::vector<char> cubin;
  return compile_cubin_locked(kron_source(words, n, M, elem, gbits, ngroups, pos, J, L, nv), cubin,
                              err) ? 0 : -1;
}

// The planned apply from a materialised map: the fused kernel's traversal and
// batching with the sources read from perm (k2[o] = k1[perm[o]]).
int jit_apply(int M, const uint8_t* sigma, uint32_t chunk_log2, int elem, const uint32_t* perm,
              const void* k1, void* k2, void* ticket, int blocks, int warps, cudaStream_t st,
              std::string& err) {
  CUfunction fn = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    if (!(g_nvrtc.ok && g_drv.ok)) {
      err = g_status;
      return -1;
    }
    const std::vector<uint32_t> keyw = gather_key(nullptr, 0, sigma, elem, warps, M);
    const uint64_t kind = 0x6170706c79ull;
    const uint64_t key = fnv(keyw.data(), (int)keyw.size(), kind);
    for (const Entry& e : g_cache[key])
      if (e.M == M && e.words == keyw) fn = e.fn;
    if (!fn)
      fn = get_kernel_locked(kind, keyw, M, fused_source(nullptr, 0, M, sigma, elem, true, warps, sigma_ident(sigma, M)),
                             "qsim_jit_apply", err);
    if (!fn) return -1;
  }
  return launch_gather(fn, M, sigma, chunk_log2, k1, k2, const_cast<uint32_t*>(perm), ticket,
                       blocks, warps, st, err);
}

int jit_local(const uint32_t* words, int n, int M, int elem, int T, const void* k1, void* k2,
              uint32_t* perm_out, int sms, cudaStream_t st, std::string& err) {
  const int smem = 2 * (elem << T);
  CUfunction fn = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    if (!(g_nvrtc.ok && g_drv.ok)) {
      err = g_status;
      return -1;
    }
    std::vector<uint32_t> keyw(words, words + n);
    keyw.push_back((uint32_t)elem);
    keyw.push_back((uint32_t)T);
    const uint64_t kind = 0x6c6f63616cull;
    const uint64_t key = fnv(keyw.data(), (int)keyw.size(), kind);
    for (const Entry& e : g_cache[key])
      if (e.M == M && e.words == keyw) fn = e.fn;
    if (!fn) {
      fn = get_kernel_locked(kind, keyw, M, local_source(words, n, M, elem, T), "qsim_jit_local", err);
      if (!fn) return -1;
      if (g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem) != CUDA_SUCCESS) {
        err = "cuFuncSetAttribute(max dynamic smem) failed";
        return -1;
      }
      g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 100);
    }
  }
  uint64_t ntiles = (1ull << M) >> T;
  uint64_t blocks = (uint64_t)sms;
  if (blocks > ntiles) blocks = ntiles;
  void* args[] = {&ntiles, const_cast<void**>(&k1), &k2, &perm_out};
  if (g_drv.launch(fn, (unsigned)blocks, 1, 1, 256, 1, 1, (unsigned)smem, (CUstream)st, args,
                   nullptr) != CUDA_SUCCESS) {
    err = "cuLaunchKernel failed";
    return -1;
  }
  return 0;
}

int jit_check_compile_local(const uint32_t* words, int n, int M, int elem, int T, std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  if (!g_nvrtc.ok) {
    err = g_status;
    return -1;
  }
  std::vector<char> cubin;
  return compile_cubin_locked(local_source(words, n, M, elem, T), cubin, err) ? 0 : -1;
}

int jit_check_compile_apply(int M, const uint8_t* sigma, int elem, std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  if (!g_nvrtc.ok) {
    err = g_status;
    return -1;
  }
  std::vector<char> cubin;
  return compile_cubin_locked(fused_source(nullptr, 0, M, sigma, elem, true, 8, sigma_ident(sigma, M)), cubin, err) ? 0 : -1;
}

int jit_check_compile_fused(const uint32_t* words, int n, int M, const uint8_t* sigma, int elem,
                            std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  if (!g_nvrtc.ok) {
    err = g_status;
    return -1;
  }
  std::vector<char> cubin;
  return compile_cubin_locked(fused_source(words, n, M, sigma, elem, false, 8, sigma_ident(sigma, M)), cubin, err) ? 0 : -1;
}

}  // namespace qsim
