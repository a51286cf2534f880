// qsim_api.cu -- the C ABI declared in include/qsim.h: argument validation,
// gate packing into the kernel-parameter bank, traversal plans, launch
// configuration.
//
// The host never computes outputs: every step of the path (the address walk
// and the gather) runs in the kernels of qsim_kernels.cuh.  The only host
// arithmetic is packing the gate list and, in qsim_plan_create, sampling the
// circuit to choose a traversal order.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "qsim.h"
#include "qsim_jit.h"
#include "qsim_kernels.cuh"

namespace {

thread_local char g_err[512] = "";
constexpr uint64_t kJitMinCount = 1ull << 22;  // outputs from which AUTO uses the JIT kernels
thread_local int32_t g_launches = 0;
thread_local const char* g_last_kernel = "";

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
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      n = v;
    else
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

int check_gates_args(const qsim_gate* gates, int32_t n, int32_t M) {
  if (M < 1 || M > 32) return QSIM_ERANGE;
  if (n < 0 || n > QSIM_MAX_GATES) return QSIM_ECAP;
  if (n > 0 && gates == nullptr) return QSIM_EINVAL;
  return QSIM_OK;
}

// Controls a kind uses (the "other bit" for SWAP counts as one).
int gate_nctrl(uint8_t kind) { return kind == 6 ? 1 : kind % 3; }

// Validate one gate (P:L43 step semantics; readings R3-R5, R17).
int check_gate(const qsim_gate& g, int32_t M) {
  if (g.kind > 6) return QSIM_EINVAL;
  const int nc = gate_nctrl(g.kind);
  if (g.target >= M) return QSIM_EBIT;
  if (nc >= 1 && (g.c0 >= M || g.c0 == g.target)) return QSIM_EBIT;
  if (nc == 2 && (g.c1 >= M || g.c1 == g.target || g.c1 == g.c0)) return QSIM_EBIT;
  return QSIM_OK;
}

// Any phase step (Z, CZ, CCZ): rows take values -1, a uint32 map alone does
// not hold the operator (qsim_build_map_signed does).
bool has_phase(const qsim_gate* gates, int32_t n) {
  for (int32_t k = 0; k < n; ++k)
    if (gates[k].kind >= 3 && gates[k].kind <= 5) return true;
  return false;
}

int check_gates(const qsim_gate* gates, int32_t n, int32_t M) {
  int rc = check_gates_args(gates, n, M);
  for (int32_t k = 0; rc == QSIM_OK && k < n; ++k) rc = check_gate(gates[k], M);
  return rc;
}

// The input-on-the-fly path takes M up to 63 (64-bit addresses).
int check_gates_kron(const qsim_gate* gates, int32_t n, int32_t M) {
  if (M < 1 || M > 63) return QSIM_ERANGE;
  if (n < 0 || n > QSIM_MAX_GATES) return QSIM_ECAP;
  if (n > 0 && gates == nullptr) return QSIM_EINVAL;
  int rc = QSIM_OK;
  for (int32_t k = 0; rc == QSIM_OK && k < n; ++k) rc = check_gate(gates[k], M);
  return rc;
}

// Pack for the kernels (gates already validated).  bitsliced: target |
// c0 << 8 | c1 << 16 | op << 24 with absent controls = the all-ones plane
// (op: toggle / swap / phase); per-lane (and NVRTC): kind | target << 8 |
// c0 << 16 | c1 << 24 with absent controls = 0.
template <int CAP>
void pack_gates(const qsim_gate* gates, int32_t n, bool bitsliced, qsim::GateList<CAP>& out) {
  out.n = (uint32_t)n;
  for (int32_t k = 0; k < n; ++k) {
    const qsim_gate& g = gates[k];
    const int nc = gate_nctrl(g.kind);
    if (bitsliced) {
      const uint32_t c0 = nc >= 1 ? g.c0 : qsim::kOnesPlane;
      const uint32_t c1 = nc == 2 ? g.c1 : qsim::kOnesPlane;
      const uint32_t op = g.kind == 6 ? qsim::kOpSwap : g.kind >= 3 ? qsim::kOpPhase : qsim::kOpToggle;
      out.w[k] = (uint32_t)g.target | (c0 << 8) | (c1 << 16) | (op << 24);
    } else {
      const uint32_t c0 = nc >= 1 ? g.c0 : 0u, c1 = nc == 2 ? g.c1 : 0u;
      out.w[k] = (uint32_t)g.kind | ((uint32_t)g.target << 8) | (c0 << 16) | (c1 << 24);
    }
  }
}

int check_range(int32_t M, uint64_t start, uint64_t count) {
  const uint64_t N = 1ull << M;
  if (start > N || count > N - start) return QSIM_ERANGE;
  return QSIM_OK;
}

qsim::SigmaParams identity_sigma(int32_t M) {
  qsim::SigmaParams sp;
  for (int k = 0; k < 32; ++k) sp.sigma[k] = (uint8_t)k;
  sp.chunk_log2 = 10;
  sp.nbits = (uint32_t)M;
  sp.ticket = nullptr;
  return sp;
}

// Natural-order walk over [start, start+count): MODE 0 writes perm_out,
// MODE 1 gathers k1 into k2_out (fused).
template <int CAP, int MODE, typename T>
int launch_walk_cap(const qsim_gate* gates, int32_t n, int32_t M, uint64_t start, uint64_t count,
                    uint32_t* perm_out, const T* k1, T* k2_out, int32_t walk, cudaStream_t st,
                    uint32_t* signs_out) {
  if (count == 0) return QSIM_OK;
  const int sms = sm_count();
  std::unique_ptr<qsim::GateList<CAP>> gl(new qsim::GateList<CAP>);
  if (walk == QSIM_WALK_PER_LANE) {
    pack_gates<CAP>(gates, n, false, *gl);
    constexpr int APT = 4;
    const uint64_t threads = (count + APT - 1) / APT;
    uint64_t blocks = (threads + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8 * 16;
    if (blocks > cap) blocks = cap;
    qsim::k_walk_per_lane<CAP, MODE, T, APT><<<(unsigned)blocks, 256, 0, st>>>(
        *gl, start, count, perm_out, k1, k2_out);
    QSIM_CHECK_LAUNCH("k_walk_per_lane");
    return QSIM_OK;
  }
  pack_gates<CAP>(gates, n, true, *gl);
  const qsim::SigmaParams sp = identity_sigma(M);
  const uint64_t tb = start >> 10, te = (start + count + 1023) >> 10;
  uint64_t blocks = (te - tb + qsim::kBsWarps - 1) / qsim::kBsWarps;
  const uint64_t cap = (uint64_t)sms * 2 * 16;
  if (blocks > cap) blocks = cap;
  const size_t smem = qsim::bs_smem_bytes((uint32_t)n);
  if (MODE == 0) {
    cudaFuncSetAttribute(qsim::k_build_bitsliced<CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    qsim::k_build_bitsliced<CAP><<<(unsigned)blocks, qsim::kBsThreads, smem, st>>>(
        *gl, sp, start, start + count, tb, te, perm_out, signs_out);
    QSIM_CHECK_LAUNCH("k_build_bitsliced");
  } else {
    cudaFuncSetAttribute(qsim::k_fused_bitsliced<CAP, T>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qsim::k_fused_bitsliced<CAP, T><<<(unsigned)blocks, qsim::kBsThreads, smem, st>>>(
        *gl, sp, start, start + count, tb, te, k1, k2_out);
    QSIM_CHECK_LAUNCH("k_fused_bitsliced");
  }
  return QSIM_OK;
}

template <int MODE, typename T>
int launch_walk(const qsim_gate* gates, int32_t n, int32_t M, uint64_t start, uint64_t count,
                uint32_t* perm_out, const T* k1, T* k2_out, int32_t walk, cudaStream_t st,
                uint32_t* signs_out = nullptr) {
  if (n <= 64)
    return launch_walk_cap<64, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out, walk, st,
                                        signs_out);
  if (n <= 256)
    return launch_walk_cap<256, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out, walk, st,
                                         signs_out);
  if (n <= 1024)
    return launch_walk_cap<1024, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out, walk,
                                          st, signs_out);
  return launch_walk_cap<qsim::kMaxGates, MODE, T>(gates, n, M, start, count, perm_out, k1, k2_out,
                                                   walk, st, signs_out);
}

// Large builds use the circuit-specialised kernel (qsim_jit.cu) when NVRTC
// is present; everything else (and any JIT failure under AUTO) uses the
// shared-memory bit-sliced interpreter (kJitMinCount, top of file).

// ---- In-thread output bits (the NVRTC build and on-the-fly input kernels)
// Each NVRTC thread holds 32 outputs that differ in 5 output bits J (the bit
// positions of its planes; lanes are output bits 0..4).  When the sources of
// those 32 outputs differ only in a few address bits V, the kernels form
// everything that depends on the other bits once per thread.  J is chosen
// greedily from sampled single-bit influences (flip output bit j, see which
// source bits change), then V is measured on all 32 combinations of the
// chosen bits.  A sample can miss a rare influence: the kernels check per
// warp tile and take the general path there (same bytes).  Host arithmetic
// only samples the circuit.
struct ThreadBits {
  uint8_t J[5];
  int L;                    // tiles fill aligned blocks of 2^L outputs
  uint64_t V;               // 0: no fast path
  std::vector<uint64_t> xs, s0;  // the sample (outputs, their sources)
};

// source address of output x (the walk, gates last to first; phase steps do
// not move addresses)
uint64_t walk_src(const qsim_gate* g, int n, uint64_t x) {
  for (int k = n - 1; k >= 0; --k) {
    const qsim_gate& q = g[k];
    const uint64_t tm = 1ull << q.target;
    if (q.kind == 6) {
      if (((x >> q.target) ^ (x >> q.c0)) & 1ull) x ^= tm | (1ull << q.c0);
      continue;
    }
    if (q.kind >= 3) continue;
    const uint64_t cm = (q.kind >= 1 ? 1ull << q.c0 : 0ull) | (q.kind == 2 ? 1ull << q.c1 : 0ull);
    if ((~x & cm) == 0ull) x ^= tm;
  }
  return x;
}

// Blocks of 2^L outputs hold whole tiles: a range that is not aligned to
// them computes part of its first and last block for nothing -- allow that
// up to 1/8 of the count.  Returns L (10 when no larger block fits).
int range_block_bits(int M, uint64_t start, uint64_t count) {
  const uint64_t end = start + count;
  int L = M;
  auto ok = [&](int l) {
    const uint64_t B = 1ull << l, m = B - 1;
    return ((start & m) == 0 && (end & m) == 0) || (B <= count / 16);
  };
  while (L > 10 && !ok(L)) --L;
  return L;
}

// jmax: in-thread bits are chosen below min(L, jmax)
void thread_bits(const qsim_gate* g, int n, int M, uint64_t start, uint64_t count, int maxv,
                 bool require_affine, ThreadBits* tb, int jmax = 64, bool store_order = false) {
  for (int k = 0; k < 5; ++k) tb->J[k] = (uint8_t)(5 + k);
  tb->L = 10;
  tb->V = 0;
  const char* env = std::getenv("QSIM_THREAD_BITS");  // A/B switch
  // from the count where AUTO takes the NVRTC kernels: below it the
  // ahead-of-time kernels run, which would pay a per-entry bit permutation
  if ((env && env[0] == '0') || M < 12 || count < kJitMinCount) return;
  const int L = range_block_bits(M, start, count);
  if (L <= 10) return;
  const int jtop = std::min(L, jmax);
  if (jtop < 10) return;
  uint64_t h = 0x9e3779b97f4a7c15ull ^ ((uint64_t)M << 32) ^ (uint64_t)n;
  auto next = [&]() {  // splitmix64
    uint64_t z = (h += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  int S = n > 1024 ? 16 : 64;
  if (const char* se = std::getenv("QSIM_THREAD_BITS_SAMPLES")) S = std::max(1, std::atoi(se));  // tests
  tb->xs.resize(S);
  tb->s0.resize(S);
  for (int i = 0; i < S; ++i) {
    tb->xs[i] = start + next() % count;
    tb->s0[i] = walk_src(g, n, tb->xs[i]);
  }
  uint64_t infl[64] = {0};
  for (int j = 5; j < jtop; ++j)
    for (int i = 0; i < S; ++i) infl[j] |= tb->s0[i] ^ walk_src(g, n, tb->xs[i] ^ (1ull << j));
  uint64_t V = 0, Jm = 0;
  int J[5];
  for (int k = 0; k < 5; ++k) {
    int best = -1, bc = 99;
    for (int j = 5; j < jtop; ++j) {
      if ((Jm >> j) & 1ull) continue;
      const int c = __builtin_popcountll(V | infl[j]);
      if (c < bc) bc = c, best = j;
    }
    J[k] = best;
    Jm |= 1ull << best;
    V |= infl[best];
  }
  if (store_order) {
    // the on-the-fly input is bound by its store pattern: every 5-subset of
    // in-thread bits whose sources vary in at most maxv bits, preferring one
    // that holds output bit 6 (then 7), then the fewest varying bits, then
    // the lowest bits.  The stores alone (tools/mb/mb_store_kron.cu): J with
    // bit 6 -- 6.7.8.13.26, 6.7.26.29.30 -- 5.00 ms like J = 5..9, J without
    // it 5.18-5.26 ms (profiles/r02_mb_store_kron_j.jsonl); the kernel:
    // cfg5 5.35 -> 5.15 ms, the M = 40 portion 5.36 -> 5.19 ms
    // (profiles/r02_kron_j_ab.txt)
    long best_key = -1;
    int bj[5] = {0, 0, 0, 0, 0};
    const int lo = 5, hi = jtop;
    for (int a = lo; a < hi; ++a)
      for (int b = a + 1; b < hi; ++b)
        for (int c = b + 1; c < hi; ++c) {
          const uint64_t vabc = infl[a] | infl[b] | infl[c];
          if (__builtin_popcountll(vabc) > maxv) continue;
          for (int d = c + 1; d < hi; ++d) {
            const uint64_t vabcd = vabc | infl[d];
            if (__builtin_popcountll(vabcd) > maxv) continue;
            for (int e = d + 1; e < hi; ++e) {
              const int nv = __builtin_popcountll(vabcd | infl[e]);
              if (nv > maxv) continue;
              const uint64_t jm = (1ull << a) | (1ull << b) | (1ull << c) | (1ull << d) | (1ull << e);
              const long key = ((long)(!((jm >> 6) & 1ull)) << 40) | ((long)(!((jm >> 7) & 1ull)) << 32) |
                               ((long)nv << 16) | (long)(a + b + c + d + e);
              if (best_key < 0 || key < best_key) {
                best_key = key;
                bj[0] = a, bj[1] = b, bj[2] = c, bj[3] = d, bj[4] = e;
              }
            }
          }
        }
    if (best_key >= 0) {
      V = 0;
      for (int k = 0; k < 5; ++k) {
        J[k] = bj[k];
        V |= infl[bj[k]];
      }
    }
  }
  std::sort(J, J + 5);
  V = 0;
  int nonaffine = 0;  // samples whose 32 sources are not s0 ^ (a XOR of 5 columns)
  for (int i = 0; i < S; ++i) {
    const uint64_t b0 = tb->xs[i] & ~Jm;
    uint64_t sc[32];
    for (int c = 0; c < 32; ++c) {
      uint64_t x = b0;
      for (int k = 0; k < 5; ++k)
        if ((c >> k) & 1) x |= 1ull << J[k];
      sc[c] = walk_src(g, n, x);
      V |= sc[0] ^ sc[c];
    }
    bool aff = true;
    for (int c = 1; c < 32 && aff; ++c) {
      uint64_t lin = sc[0];
      for (int k = 0; k < 5; ++k)
        if ((c >> k) & 1) lin ^= sc[0] ^ sc[1 << k];
      aff = lin == sc[c];
    }
    nonaffine += !aff;
  }
  const int nv = __builtin_popcountll(V);
  if (nv == 0 || nv > maxv) return;
  if (require_affine && nonaffine * 16 > S) return;  // the affine fast path would mostly fail
  // the kernels check per warp (32 threads = output bits 0..4): one thread
  // whose bits outside V move, or (build) whose sources are not affine in J,
  // sends the whole warp tile down the general path -- sample whole warps
  const int W = n > 1024 ? 4 : 16;
  int failed = 0;
  for (int w = 0; w < W; ++w) {
    const uint64_t b0 = (start + next() % count) & ~Jm & ~31ull;
    bool ok = true;
    for (uint64_t lane = 0; lane < 32 && ok; ++lane) {
      uint64_t sc[32];
      for (int c = 0; c < 32; ++c) {
        uint64_t x = b0 | lane;
        for (int k = 0; k < 5; ++k)
          if ((c >> k) & 1) x |= 1ull << J[k];
        sc[c] = walk_src(g, n, x);
        ok = ok && ((sc[0] ^ sc[c]) & ~V) == 0;
      }
      for (int c = 1; c < 32 && ok && require_affine; ++c) {
        uint64_t lin = sc[0];
        for (int k = 0; k < 5; ++k)
          if ((c >> k) & 1) lin ^= sc[0] ^ sc[1 << k];
        ok = lin == sc[c];
      }
    }
    failed += !ok;
  }
  if (failed * 8 > W) return;  // more than 1 in 8 warp tiles would take the general path
  for (int k = 0; k < 5; ++k) tb->J[k] = (uint8_t)J[k];
  tb->L = L;
  tb->V = V;
}

// one-entry caches: repeated calls on the same circuit and range (a bench
// loop, a batch) sample once
struct ThreadBitsCache {
  std::mutex mu;
  std::vector<qsim_gate> gates;
  std::string env;
  int M = -1, maxv = 0;
  uint64_t start = 0, count = 0;
  ThreadBits tb;
};
ThreadBitsCache g_tb_cache[2];  // 0: build, 1: on-the-fly input

void thread_bits_cached(int which, const qsim_gate* g, int n, int M, uint64_t start, uint64_t count,
                        int maxv, ThreadBits* tb) {
  ThreadBitsCache& c = g_tb_cache[which];
  std::lock_guard<std::mutex> lk(c.mu);
  const char* e1 = std::getenv("QSIM_THREAD_BITS");
  const char* e2 = std::getenv("QSIM_THREAD_BITS_SAMPLES");
  const std::string env = std::string(e1 ? e1 : "-") + "/" + (e2 ? e2 : "-");
  const bool hit = c.env == env && c.M == M && c.maxv == maxv && c.start == start &&
                   c.count == count && c.gates.size() == (size_t)n &&
                   (n == 0 || std::memcmp(c.gates.data(), g, sizeof(qsim_gate) * n) == 0);
  if (!hit) {
    thread_bits(g, n, M, start, count, maxv, which == 0, &c.tb);
    c.gates.assign(g, g + n);
    c.env = env;
    c.M = M, c.maxv = maxv, c.start = start, c.count = count;
  }
  *tb = c.tb;
}

// On-the-fly input: the table layout.  Table 0 (one lookup per entry) is
// indexed by V and gb - |V| more bits the lanes (output bits 0..4) do not
// move, so that the 32 lanes of a warp read few distinct entries of table 0
// (a broadcast rather than bank conflicts); the other groups' product is
// formed once per thread.
struct KronLayout {
  uint8_t pos[64];
  uint8_t J[5];
  int L, nv;
};

// The table grouping decides the rounding of every entry, so it depends on
// the circuit alone (never on the range or the call history): the in-thread
// bits J and the varying source bits V are sampled once over the whole
// output space [0, 2^M) with a fixed seed -- output portions then glue byte
// for byte.  J is chosen below bit 28 when M > 32 (so 2^32-entry portions
// aligned to 2^28 can use it).  The traversal of a range uses the circuit's J
// when its blocks hold them (L > max J), else the default J and the general
// path (same tables, same products, same bytes).
void kron_layout(const qsim_gate* g, int n, int M, int gb, int ng, uint64_t start, uint64_t count,
                 bool jit, KronLayout* ly) {
  for (int k = 0; k < 64; ++k) ly->pos[k] = (uint8_t)k;
  for (int k = 0; k < 5; ++k) ly->J[k] = (uint8_t)(5 + k);
  ly->L = 10;
  ly->nv = 0;
  if (ng < 2) return;
  ThreadBits tb;
  {
    ThreadBitsCache& c = g_tb_cache[1];
    std::lock_guard<std::mutex> lk(c.mu);
    const char* e1 = std::getenv("QSIM_THREAD_BITS");
    const char* e2 = std::getenv("QSIM_THREAD_BITS_SAMPLES");
    const std::string env = std::string(e1 ? e1 : "-") + "/" + (e2 ? e2 : "-");
    const bool hit = c.env == env && c.M == M && c.maxv == gb && c.gates.size() == (size_t)n &&
                     (n == 0 || std::memcmp(c.gates.data(), g, sizeof(qsim_gate) * n) == 0);
    if (!hit) {
      thread_bits(g, n, M, 0, 1ull << M, gb, false, &c.tb, M > 32 ? 28 : 64, true);
      c.gates.assign(g, g + n);
      c.env = env;
      c.M = M, c.maxv = gb, c.start = 0, c.count = 1ull << M;
    }
    tb = c.tb;
  }
  const uint64_t V = tb.V;
  if (!V) return;
  uint64_t lanes = 0;
  for (int j = 0; j < 5; ++j)
    for (size_t i = 0; i < tb.xs.size(); ++i) lanes |= tb.s0[i] ^ walk_src(g, n, tb.xs[i] ^ (1ull << j));
  uint64_t G0 = V;
  for (int pass = 0; pass < 2; ++pass)
    for (int b = M - 1; b >= 0 && __builtin_popcountll(G0) < gb; --b)
      if (!((G0 >> b) & 1ull) && (pass == 1 || !((lanes >> b) & 1ull))) G0 |= 1ull << b;
  int k = 0;
  for (int b = 0; b < M; ++b)
    if ((V >> b) & 1ull) ly->pos[k++] = (uint8_t)b;
  for (int b = 0; b < M; ++b)
    if (((G0 & ~V) >> b) & 1ull) ly->pos[k++] = (uint8_t)b;
  for (int b = 0; b < M; ++b)
    if (!((G0 >> b) & 1ull)) ly->pos[k++] = (uint8_t)b;
  // the range's traversal (speed only)
  if (!jit || count < kJitMinCount) return;
  const int L = range_block_bits(M, start, count);
  int jhi = 0;
  for (int j = 0; j < 5; ++j) jhi = std::max(jhi, (int)tb.J[j]);
  if (L <= 10 || jhi >= L) return;
  for (int j = 0; j < 5; ++j) ly->J[j] = tb.J[j];
  ly->L = L;
  ly->nv = __builtin_popcountll(V);
}

// build kernel fast path up to this many varying address bits per thread
// (each costs ~27 ops per thread; measured: |V| <= 6 faster, 8 neutral to slower)
constexpr int kBuildMaxV = 6;
thread_local char g_build_name[96];

int build_impl(const qsim_gate* gates, int32_t n, int32_t M, uint64_t start, uint64_t count,
               uint32_t* perm_out, int32_t walk, cudaStream_t st) {
  g_last_kernel = "";
  int rc = check_gates(gates, n, M);
  if (rc) return rc;
  if (has_phase(gates, n)) {  // the map alone would drop the -1 rows
    std::snprintf(g_err, sizeof g_err, "phase gates: use qsim_build_map_signed");
    return QSIM_EINVAL;
  }
  if ((rc = check_range(M, start, count))) return rc;
  if (walk < 0 || walk > 3) return QSIM_EINVAL;
  if (perm_out == nullptr || !aligned16(perm_out)) return QSIM_EINVAL;
  if (walk == QSIM_WALK_JIT || (walk == QSIM_WALK_AUTO && count >= kJitMinCount)) {
    std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
    pack_gates(gates, n, false, *gl);
    std::string err;
    ThreadBits tb;  // in-thread affine fast path (QSIM_BUILD_THREAD_BITS=0: J = 5..9, transpose)
    const char* bt = std::getenv("QSIM_BUILD_THREAD_BITS");
    thread_bits_cached(0, gates, n, M, start, (bt && bt[0] == '0') ? 0 : count, kBuildMaxV, &tb);
    if (qsim::jit_build(gl->w, n, M, tb.J, tb.L, tb.V, start, count, perm_out, sm_count(), st,
                        err) == 0) {
      if (count) ++g_launches;
      std::snprintf(g_build_name, sizeof g_build_name, "qsim_jit_build (J %d.%d.%d.%d.%d, L %d, nv %d)",
                    tb.J[0], tb.J[1], tb.J[2], tb.J[3], tb.J[4], tb.L, __builtin_popcountll(tb.V));
      g_last_kernel = g_build_name;
      return QSIM_OK;
    }
    if (walk == QSIM_WALK_JIT) {
      std::snprintf(g_err, sizeof g_err, "jit: %s", err.c_str());
      return QSIM_ECUDA;
    }
    walk = QSIM_WALK_BITSLICED;
  }
  return launch_walk<0, uint2>(gates, n, M, start, count, perm_out, nullptr, nullptr, walk, st);
}

// Phased permutation, materialised: perm and the row values (signs bitmap),
// natural order, bit-sliced walk (the sign plane rides along).
int build_signed_impl(const qsim_gate* gates, int32_t n, int32_t M, uint64_t start, uint64_t count,
                      uint32_t* perm_out, uint32_t* signs_out, cudaStream_t st) {
  int rc = check_gates(gates, n, M);
  if (rc) return rc;
  if ((rc = check_range(M, start, count))) return rc;
  if (start % 32) return QSIM_EINVAL;
  if (!perm_out || !signs_out || !aligned16(perm_out) || (reinterpret_cast<uintptr_t>(signs_out) & 3u))
    return QSIM_EINVAL;
  if (overlap(perm_out, count * 4, signs_out, (count + 31) / 32 * 4)) return QSIM_EALIAS;
  return launch_walk<0, uint2>(gates, n, M, start, count, perm_out, nullptr, nullptr,
                               QSIM_WALK_BITSLICED, st, signs_out);
}

int apply_signed_impl(const uint32_t* perm, const uint32_t* signs, uint64_t count, int32_t M,
                      int32_t dtype, const void* k1, void* k2, cudaStream_t st) {
  if (M < 1 || M > 32) return QSIM_ERANGE;
  if (count > (1ull << M)) return QSIM_ERANGE;
  const int e = elem_bytes(dtype);
  if (e == 0) return QSIM_EINVAL;
  if (!perm || !signs || !k1 || !k2 || !aligned16(perm) || !aligned16(k1) || !aligned16(k2) ||
      (reinterpret_cast<uintptr_t>(signs) & 3u))
    return QSIM_EINVAL;
  const uint64_t N = 1ull << M;
  if (overlap(k1, N * e, k2, count * e) || overlap(perm, count * 4, k2, count * e) ||
      overlap(signs, (count + 31) / 32 * 4, k2, count * e))
    return QSIM_EALIAS;
  if (count == 0) return QSIM_OK;
  uint64_t blocks = (count / 4 + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * 8 * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  if (dtype == QSIM_C64)
    qsim::k_apply_signed<uint2><<<(unsigned)blocks, 256, 0, st>>>(
        perm, signs, count, static_cast<const uint2*>(k1), static_cast<uint2*>(k2));
  else
    qsim::k_apply_signed<uint4><<<(unsigned)blocks, 256, 0, st>>>(
        perm, signs, count, static_cast<const uint4*>(k1), static_cast<uint4*>(k2));
  QSIM_CHECK_LAUNCH("k_apply_signed");
  return QSIM_OK;
}

int fused_impl(const qsim_gate* gates, int32_t n, int32_t M, int32_t dtype, uint64_t start,
               uint64_t count, const void* k1, void* k2, int32_t walk, cudaStream_t st) {
  int rc = check_gates(gates, n, M);
  if (rc) return rc;
  if ((rc = check_range(M, start, count))) return rc;
  if (walk < 0 || walk > 2) return QSIM_EINVAL;
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

// ---- Appendix 1: input generated on the fly, fused with the map
// Product-table groups: as few groups (complex products per entry + 1) as fit
// tables of <= 2^10 complex64 / 2^8 complex128 entries.  Measured
// (profiles/r01_kron_group_bits.txt): M = 40 complex64 4 groups of 10 bits
// 11.96 ms vs 5 bytes 14.6 ms; M = 32 4 bytes 9.22 ms vs 3 groups of 11 bits
// 11.7 ms (larger tables cost more than the product they save).
void kron_groups(int32_t M, int e, uint32_t* gbits, uint32_t* ngroups) {
  int maxb = e == 8 ? 10 : 8;
  const int ng = (M + maxb - 1) / maxb;
  *ngroups = (uint32_t)ng;
  *gbits = (uint32_t)((M + ng - 1) / ng);
}

thread_local char g_kron_name[96];

template <int CAP, typename C>
int launch_kron_cap(const qsim_gate* gates, int32_t n, int32_t M, const qsim::Qubits& qb,
                    uint64_t start, uint64_t count, C* k2, cudaStream_t st) {
  std::unique_ptr<qsim::GateList<CAP>> gl(new qsim::GateList<CAP>);
  pack_gates<CAP>(gates, n, true, *gl);
  const qsim::SigmaParams sp = identity_sigma(M);
  const uint64_t tb = start >> 10, te = (start + count + 1023) >> 10;
  uint64_t blocks = (te - tb + qsim::kBsWarps - 1) / qsim::kBsWarps;
  const uint64_t cap = (uint64_t)sm_count() * 2 * 16;
  if (blocks > cap) blocks = cap;
  const size_t smem = ((qsim::bs_smem_bytes((uint32_t)n) + 15) & ~(size_t)15) +
                      qsim::kron_table_bytes(qb.gbits, qb.ngroups, sizeof(C));
  cudaFuncSetAttribute(qsim::k_fused_kron_bitsliced<CAP, C>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  qsim::k_fused_kron_bitsliced<CAP, C><<<(unsigned)blocks, qsim::kBsThreads, smem, st>>>(
      *gl, sp, qb, start, start + count, tb, te, k2);
  QSIM_CHECK_LAUNCH("k_fused_kron_bitsliced");
  return QSIM_OK;
}

template <typename C>
int launch_kron(const qsim_gate* gates, int32_t n, int32_t M, const qsim::Qubits& qb,
                uint64_t start, uint64_t count, C* k2, cudaStream_t st) {
  if (n <= 64) return launch_kron_cap<64, C>(gates, n, M, qb, start, count, k2, st);
  if (n <= 256) return launch_kron_cap<256, C>(gates, n, M, qb, start, count, k2, st);
  if (n <= 1024) return launch_kron_cap<1024, C>(gates, n, M, qb, start, count, k2, st);
  return launch_kron_cap<qsim::kMaxGates, C>(gates, n, M, qb, start, count, k2, st);
}

template <typename C>
int launch_kron64(const qsim_gate* gates, int32_t n, const qsim::Qubits& qb, uint64_t start,
                  uint64_t count, C* k2, cudaStream_t st) {
  std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
  pack_gates(gates, n, false, *gl);
  uint64_t blocks = (count + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  const size_t smem = qsim::kron_table_bytes(qb.gbits, qb.ngroups, sizeof(C));
  cudaFuncSetAttribute(qsim::k_fused_kron_perlane64<qsim::kMaxGates, C>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  qsim::k_fused_kron_perlane64<qsim::kMaxGates, C><<<(unsigned)blocks, 256, smem, st>>>(
      *gl, qb, start, count, k2);
  QSIM_CHECK_LAUNCH("k_fused_kron_perlane64");
  return QSIM_OK;
}

int kron_impl(const qsim_gate* gates, int32_t n, int32_t M, int32_t dtype, const double* qubits,
              uint64_t start, uint64_t count, void* k2, int32_t walk, cudaStream_t st) {
  // M up to 63 here (64-bit addresses): k1 is generated, never stored
  int rc = check_gates_kron(gates, n, M);
  if (rc) return rc;
  if ((rc = check_range(M, start, count))) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0 || !qubits || !k2 || !aligned16(k2)) return QSIM_EINVAL;
  if (walk < QSIM_WALK_AUTO || walk > QSIM_WALK_JIT) return QSIM_EINVAL;
  qsim::Qubits qb;
  std::memset(&qb, 0, sizeof qb);
  qb.M = (uint32_t)M;
  kron_groups(M, e, &qb.gbits, &qb.ngroups);
  for (int j = 0; j < M; ++j)
    for (int c = 0; c < 4; ++c) qb.v[j][c] = qubits[4 * j + c];
  if (count == 0) return QSIM_OK;
  KronLayout ly;  // the table grouping is the circuit's (same bytes for every range and kernel)
  kron_layout(gates, n, M, (int)qb.gbits, (int)qb.ngroups, start, count, qsim::jit_available(), &ly);
  for (int k = 0; k < 64; ++k) {
    qb.pos[k] = ly.pos[k];
    if (ly.pos[k] != k) qb.permuted = 1;
  }
  const bool jit_try = walk == QSIM_WALK_JIT ||
                       (walk == QSIM_WALK_AUTO && (M > 32 || count >= kJitMinCount));
  if (jit_try) {
    std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
    pack_gates(gates, n, false, *gl);
    std::string err;
    if (qsim::jit_kron(gl->w, n, M, &qb, sizeof qb, e, (int)qb.gbits, (int)qb.ngroups, ly.pos, ly.J,
                       ly.L, ly.nv, start, count, k2, sm_count(), st, err) == 0) {
      ++g_launches;
      std::snprintf(g_kron_name, sizeof g_kron_name, "qsim_jit_kron (J %d.%d.%d.%d.%d, L %d, nv %d)",
                    ly.J[0], ly.J[1], ly.J[2], ly.J[3], ly.J[4], ly.L, ly.nv);
      g_last_kernel = g_kron_name;
      return QSIM_OK;
    }
    if (walk == QSIM_WALK_JIT) {
      std::snprintf(g_err, sizeof g_err, "jit: %s", err.c_str());
      return QSIM_ECUDA;
    }
  }
  g_last_kernel = M > 32 || walk == QSIM_WALK_PER_LANE ? "k_fused_kron_perlane64"
                                                        : "k_fused_kron_bitsliced";
  if (M > 32 || walk == QSIM_WALK_PER_LANE) {
    if (dtype == QSIM_C64)
      return launch_kron64<float2>(gates, n, qb, start, count, static_cast<float2*>(k2), st);
    return launch_kron64<double2>(gates, n, qb, start, count, static_cast<double2*>(k2), st);
  }
  if (dtype == QSIM_C64)
    return launch_kron<float2>(gates, n, M, qb, start, count, static_cast<float2*>(k2), st);
  return launch_kron<double2>(gates, n, M, qb, start, count, static_cast<double2*>(k2), st);
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
    qsim::k_apply<uint2><<<(unsigned)blocks, 256, 0, st>>>(
        perm, count, static_cast<const uint2*>(k1), static_cast<uint2*>(k2));
  else
    qsim::k_apply<uint4><<<(unsigned)blocks, 256, 0, st>>>(
        perm, count, static_cast<const uint4*>(k1), static_cast<uint4*>(k2));
  QSIM_CHECK_LAUNCH("k_apply");
  return QSIM_OK;
}

// ---- traversal plan (host analysis of the circuit; no output is computed)
uint64_t plan_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// inverse map perm^-1(j) = f_n(...f_1(j)): Step 1 first
// A step's action on addresses (host plans): toggle tm when the controls cm
// are set; a SWAP (swap = true) toggles both bits of tm when they differ;
// phase steps leave addresses unchanged (tm = 0).
struct PlanGate {
  uint32_t cm, tm;
  bool swap;
};

uint32_t plan_step(const PlanGate& g, uint32_t x) {
  if (g.swap) {
    const uint32_t b = x & g.tm;
    return (b != 0u && b != g.tm) ? x ^ g.tm : x;
  }
  return (~x & g.cm) == 0u ? x ^ g.tm : x;
}

uint32_t plan_inverse_walk(const PlanGate* g, int n, uint32_t x) {
  for (int k = 0; k < n; ++k) x = plan_step(g[k], x);
  return x;
}

// counter bits that stay output bits: 32-byte runs of k2 and perm (8
// complex64 / 2 complex128 entries: 64 / 32 bytes of k2, 32 / 8 bytes of perm)
int plan_keep_bits(int32_t dtype) { return dtype == QSIM_C64 ? 3 : 2; }

int plan_validate(const qsim_plan* p) {
  if (!p) return QSIM_EINVAL;
  if (p->M < 1 || p->M > 32) return QSIM_ERANGE;
  if (elem_bytes(p->dtype) == 0) return QSIM_EINVAL;
  uint64_t seen = 0;
  for (int k = 0; k < p->M; ++k) {
    if (p->sigma[k] >= p->M) return QSIM_EINVAL;
    seen |= 1ull << p->sigma[k];
    if (k < plan_keep_bits(p->dtype) && p->sigma[k] != k) return QSIM_EINVAL;
  }
  if (seen != ((1ull << p->M) - 1)) return QSIM_EINVAL;
  if (p->M >= 10 && (p->chunk_log2 < 10 || (int)p->chunk_log2 > p->M)) return QSIM_EINVAL;
  if (p->M >= 10 && (p->fused_chunk_log2 < 10 || (int)p->fused_chunk_log2 > p->M))
    return QSIM_EINVAL;
  if (p->blocks_per_sm < 1 || p->blocks_per_sm > 8) return QSIM_EINVAL;
  if (p->ilp != 0 && p->ilp != 8 && p->ilp != 16 && p->ilp != 32) return QSIM_EINVAL;
  if (p->cta_threads != 0 && p->cta_threads != 256 && p->cta_threads != 512 &&
      p->cta_threads != 1024)
    return QSIM_EINVAL;
  if (p->ilp == 32 && p->cta_threads == 1024) return QSIM_EINVAL;  // register file
  return QSIM_OK;
}

bool plan_natural(const qsim_plan* p) { return (p->flags & 1u) || p->M < 10; }

// warps per CTA of the NVRTC gather kernels: 16 for plans with 512-thread
// CTAs (a block of 2^14 counters per round), else 8
int jit_warps(const qsim_plan* p) { return p->cta_threads == 512 ? 16 : 8; }

// The NVRTC gather kernels take chunks from the workspace ticket in counter
// order (an in-order front: k2 / perm written close to their neighbours, k1
// lines' readers close in time).  A natural-order plan of an L2-resident
// state (<= 64 MB) gains nothing from it, and resetting the ticket costs a
// memset per call (cfg2: 14.4 -> 12.3 us per call without it); a
// natural-order plan of an HBM-resident, well-mixed state keeps it (cfg3:
// 1.50 ms with the ticket, 1.87 ms round-robin).
void* ticket_for(const qsim_plan* p, void* workspace) {
  const uint64_t bytes = (1ull << p->M) * (uint64_t)elem_bytes(p->dtype);
  return plan_natural(p) && bytes <= (64ull << 20) ? nullptr : workspace;
}

qsim::SigmaParams plan_params(const qsim_plan* p, void* workspace, bool fused = false) {
  qsim::SigmaParams sp;
  std::memcpy(sp.sigma, p->sigma, 32);
  sp.chunk_log2 = fused ? p->fused_chunk_log2 : p->chunk_log2;
  sp.nbits = (uint32_t)p->M;
  sp.ticket = static_cast<unsigned long long*>(workspace);
  return sp;
}

int reset_ticket(void* workspace, cudaStream_t st) {
  if (!workspace) return QSIM_OK;
  cudaError_t ce = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  return ce == cudaSuccess ? QSIM_OK : cuda_fail(ce, "ticket reset");
}

// A line's readers spread (max - min position of its 8 or 16 readers in a
// traversal order), as log2, 0.9-quantile over the sampled lines.
int spread_q90_log2(std::vector<uint64_t>& spreads) {
  std::sort(spreads.begin(), spreads.end());
  const uint64_t v = spreads[(spreads.size() * 9) / 10];
  int l = 0;
  while (l < 40 && (1ull << l) <= v) ++l;
  return l;
}

// perm(x) = f_1(...f_n(x)): Step n first (readings R1, R2)
uint32_t plan_forward_walk(const PlanGate* g, int n, uint32_t x) {
  for (int k = n - 1; k >= 0; --k) x = plan_step(g[k], x);
  return x;
}

// Sector cover: sample outputs i, their sources s = perm(i), and the readers
// g(s ^ r) of the other entries of s's 32-byte sector of k1 (g = perm^-1);
// the diff patterns d = g(s ^ r) ^ i say which output bits must vary within
// a block of outputs for a sector's readers to fall into it.  Greedy cover:
// start from the kept bits, repeatedly add the pattern with the best gain in
// contained pairs per added bit until T bits.  Returns the bit set V; the
// fraction of sampled pairs inside a V-block goes to plan->tile_contained.
uint32_t plan_sector_cover(const PlanGate* pg, int n, int M, int dtype, int T, qsim_plan* plan) {
  const int e = elem_bytes(dtype), keep = plan_keep_bits(dtype);
  const int eps = 32 / e;  // entries per cover granule: a 32-byte sector
  const int samples = 2048;
  std::vector<uint32_t> diffs;
  diffs.reserve((size_t)samples * (eps - 1));
  const uint64_t N = 1ull << M;
  for (int k = 0; k < samples; ++k) {
    const uint32_t i = (uint32_t)(plan_mix(0x7e57ull + k) % N);
    const uint32_t src = plan_forward_walk(pg, n, i);
    for (int r = 1; r < eps; ++r) diffs.push_back(plan_inverse_walk(pg, n, src ^ (uint32_t)r) ^ i);
  }
  std::sort(diffs.begin(), diffs.end());
  std::vector<std::pair<uint32_t, uint32_t>> pats;  // (pattern, count)
  for (size_t a = 0; a < diffs.size();) {
    size_t b = a;
    while (b < diffs.size() && diffs[b] == diffs[a]) ++b;
    pats.push_back({diffs[a], (uint32_t)(b - a)});
    a = b;
  }
  std::sort(pats.begin(), pats.end(), [](const std::pair<uint32_t, uint32_t>& x,
                                         const std::pair<uint32_t, uint32_t>& y) {
    return x.second != y.second ? x.second > y.second : x.first < y.first;
  });
  if (pats.size() > 512) pats.resize(512);  // candidates: the frequent patterns
  auto contained = [&](uint32_t V) {
    uint64_t c = 0;
    for (const auto& pc : pats)
      if ((pc.first & ~V) == 0) c += pc.second;
    return c;
  };
  const int run = keep;  // low output bits in the cover: contiguous output runs of 2^run entries
  uint32_t V = (1u << run) - 1;
  int bits = run;
  while (bits < T) {
    const uint64_t base = contained(V);
    double best = 0.0;
    uint32_t add_best = 0;
    for (const auto& pc : pats) {
      const uint32_t add = pc.first & ~V;
      const int na = __builtin_popcount(add);
      if (na == 0 || bits + na > T) continue;
      const double gain = (double)(contained(V | add) - base) / na;
      if (gain > best) {
        best = gain;
        add_best = add;
      }
    }
    if (add_best == 0) {  // no pattern fits: extend the contiguous output run
      for (int b = 0; b < M; ++b)
        if (!((V >> b) & 1u)) {
          add_best = 1u << b;
          break;
        }
    }
    V |= add_best;
    bits = __builtin_popcount(V);
  }
  uint64_t hit = 0;
  for (uint32_t d : diffs) hit += (d & ~V) == 0;
  plan->tile_contained = diffs.empty() ? 1.0f : (float)hit / (float)diffs.size();
  plan->tile_log2 = (uint8_t)T;
  return V;
}

// Cover size: the smallest T in [10, Tmax] whose greedy cover holds >= 90 %
// of the sampled pairs, else the T with the best containment (smallest on
// ties) -- cover bits beyond what the pairs need cost more than they bring
// (M = 32 seeds 4 / 7 / 8: profiles/r01_cover_size.txt).
uint32_t plan_choose_cover(const PlanGate* pg, int n, int M, int dtype, int Tmax, bool fixed,
                           qsim_plan* plan) {
  const int lo = fixed ? Tmax : std::min(10, Tmax);
  uint32_t best_v = 0;
  float best_c = -1.0f;
  int best_t = Tmax;
  for (int T = lo; T <= Tmax; ++T) {
    const uint32_t V = plan_sector_cover(pg, n, M, dtype, T, plan);
    const float c = plan->tile_contained;
    if (c >= 0.9f) {
      best_v = V;
      best_c = c;
      best_t = T;
      break;
    }
    if (c > best_c + 1e-6f) {
      best_v = V;
      best_c = c;
      best_t = T;
    }
  }
  plan->tile_contained = best_c;
  plan->tile_log2 = (uint8_t)best_t;
  return best_v;
}

// Bits the walk can change: every target, and the partner bit of a SWAP.
int moved_bits(const qsim_gate* gates, int32_t n) {
  int top = 0;
  for (int32_t k = 0; k < n; ++k) {
    top = std::max(top, (int)gates[k].target + 1);
    if (gates[k].kind == 6) top = std::max(top, (int)gates[k].c0 + 1);
  }
  return top;
}
int local_tile_bits(int32_t dtype) { return dtype == QSIM_C64 ? 13 : 12; }

// Plan construction options (qsim_plan_create uses the defaults;
// qsim_plan_tune measures variants).
struct PlanOpts {
  int cover_bits = 13;    // largest sector cover (counter bits of one L1-resident block)
  bool fixed = false;     // always cover_bits (else the smallest cover holding >= 90 %)
  bool lane_run = false;  // lanes on output bits 0..4 (bits 3, 4 added to the cover)
};

int plan_fill(const qsim_gate* gates, int32_t n, int32_t M, int32_t dtype, qsim_plan* plan,
              const PlanOpts& opts = PlanOpts()) {
  std::memset(plan, 0, sizeof *plan);
  plan->M = M;
  plan->dtype = dtype;
  // chunks: 2^15 counters (measured best on cfg5), but at least 8 chunks per SM
  int cap = M - 10 - 3;  // 2^(M-13) counters per chunk leaves >= 8 * 1024 chunks
  if (cap < 10) cap = 10;
  plan->chunk_log2 = (uint32_t)std::min(std::min(15, cap), (int)M);
  plan->fused_chunk_log2 = (uint32_t)std::min(std::min(15, cap), (int)M);
  plan->blocks_per_sm = 1;
  plan->ilp = 16;
  plan->cta_threads = 256;
  for (int k = 0; k < 32; ++k) plan->sigma[k] = (uint8_t)k;
  const int e = elem_bytes(dtype);
  if (M < 10) {
    plan->flags = 1;
    return QSIM_OK;
  }
  std::unique_ptr<PlanGate[]> pg(new PlanGate[n > 0 ? n : 1]);
  for (int k = 0; k < n; ++k) {
    const qsim_gate& g = gates[k];
    const int nc = g.kind == 6 ? 0 : g.kind % 3;
    pg[k].swap = g.kind == 6;
    pg[k].cm = (nc >= 1 ? 1u << g.c0 : 0u) | (nc == 2 ? 1u << g.c1 : 0u);
    pg[k].tm = g.kind == 6 ? (1u << g.target) | (1u << g.c0) : g.kind >= 3 ? 0u : 1u << g.target;
  }
  // one 128-byte line of k1 (wider "lines" for DRAM row locality measured
  // slower: 4/5/6/7/8 bits -> 20.0/20.1/20.6/24.1/24.0 ms on cfg5)
  const int line_bits = dtype == QSIM_C64 ? 4 : 3;
  const int lines = 2048;
  uint32_t count[32] = {0};
  const uint64_t nlines = 1ull << (M - line_bits);
  std::vector<uint32_t> readers((size_t)lines << line_bits);
  std::vector<uint64_t> spread_nat(lines);
  for (int s = 0; s < lines; ++s) {
    const uint32_t base = (uint32_t)((plan_mix(0x51a3ull + s) % nlines) << line_bits);
    uint32_t* r = &readers[(size_t)s << line_bits];
    uint32_t diff = 0, lo = 0xffffffffu, hi = 0;
    for (uint32_t d = 0; d < (1u << line_bits); ++d) {
      r[d] = plan_inverse_walk(pg.get(), n, base | d);
      diff |= r[d] ^ r[0];
      lo = std::min(lo, r[d]);
      hi = std::max(hi, r[d]);
    }
    spread_nat[s] = hi - lo;
    for (int b = 0; b < M; ++b) count[b] += (diff >> b) & 1u;
  }
  for (int b = 0; b < M; ++b) plan->change_freq[b] = (float)count[b] / lines;
  // sigma: counter bits 0..T-1 = the sector cover V (ascending: the kept bits
  // first), so the readers of a k1 sector are handled by one CTA close in time
  // (its L1 serves them); then the other bits by how often a k1 line's readers
  // differ in them (the chunk front keeps its lines in L2)
  const int T = std::max(plan_keep_bits(dtype), std::min(M, std::min(opts.cover_bits, 20)));
  uint32_t V = plan_choose_cover(pg.get(), n, M, dtype, T, opts.fixed, plan);
  if (opts.lane_run && M >= 5) V |= 31u;  // lanes on output bits 0..4: 256-byte warp stores
  int order[32], m = 0, k = 0;
  for (int b = 0; b < M; ++b) {
    if ((V >> b) & 1u)
      plan->sigma[k++] = (uint8_t)b;
    else
      order[m++] = b;
  }
  std::stable_sort(order, order + m, [&](int x, int y) { return count[x] > count[y]; });
  for (int j = 0; j < m; ++j) plan->sigma[k++] = (uint8_t)order[j];
  // spread of the readers in sigma order (counter positions)
  uint8_t inv[32];
  for (int k = 0; k < M; ++k) inv[plan->sigma[k]] = (uint8_t)k;
  std::vector<uint64_t> spread_sig(lines);
  for (int s = 0; s < lines; ++s) {
    uint64_t lo = ~0ull, hi = 0;
    for (uint32_t d = 0; d < (1u << line_bits); ++d) {
      const uint32_t r = readers[((size_t)s << line_bits) + d];
      uint64_t c = 0;
      for (int b = 0; b < M; ++b) c |= (uint64_t)((r >> b) & 1u) << inv[b];
      lo = std::min(lo, c);
      hi = std::max(hi, c);
    }
    spread_sig[s] = hi - lo;
  }
  const int nat = spread_q90_log2(spread_nat), sig = spread_q90_log2(spread_sig);
  // Natural order when the sector cover holds few sector-mate pairs (an
  // effectively random permutation, e.g. cfg3: no order helps; measured
  // equal within 5 %).
  if (plan->tile_contained < 0.25f) plan->flags = 1;
  // small states are L2-resident: natural order, full parallelism
  if ((1ull << M) * (uint64_t)e <= (64ull << 20)) plan->flags = 1;
  plan->reserved_spread = (uint16_t)(nat | (sig << 8));
  // locality-keeping circuit: every bit the walk changes lies below the tile
  if (M >= local_tile_bits(dtype) && moved_bits(gates, n) <= local_tile_bits(dtype)) plan->flags |= 2u;
  return QSIM_OK;
}

// The chunk ticket of the planned kernels when the caller passes no
// workspace (qsim_run_fused): 256 bytes per (device, stream), allocated on
// first use and kept for the process -- calls on one stream are ordered by
// the stream, so they can share it.  During stream capture nothing is
// allocated (nullptr: round-robin chunks).
std::mutex g_ticket_mu;
std::vector<std::pair<std::pair<int, cudaStream_t>, void*>> g_tickets;

void* stream_ticket(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_ticket_mu);
  for (const auto& t : g_tickets)
    if (t.first.first == dev && t.first.second == st) return t.second;
  void* p = nullptr;
  if (cudaMalloc(&p, 256) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  g_tickets.push_back({{dev, st}, p});
  return p;
}

// Plans of recent circuits (qsim_run_fused, qsim_run_host*): the host
// sampling runs once per (circuit, M, dtype); a few entries, most recent first.
struct PlanCacheEntry {
  std::vector<qsim_gate> gates;
  int32_t M, dtype;
  qsim_plan plan;
};
std::mutex g_plan_mu;
std::vector<PlanCacheEntry> g_plan_cache;

int cached_plan(const qsim_gate* gates, int32_t n, int32_t M, int32_t dtype, qsim_plan* out) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (size_t i = 0; i < g_plan_cache.size(); ++i) {
    const PlanCacheEntry& c = g_plan_cache[i];
    if (c.M == M && c.dtype == dtype && c.gates.size() == (size_t)n &&
        (n == 0 || std::memcmp(c.gates.data(), gates, sizeof(qsim_gate) * n) == 0)) {
      *out = c.plan;
      std::rotate(g_plan_cache.begin(), g_plan_cache.begin() + i, g_plan_cache.begin() + i + 1);
      return QSIM_OK;
    }
  }
  PlanCacheEntry c;
  int rc = plan_fill(gates, n, M, dtype, &c.plan);
  if (rc) return rc;
  c.gates.assign(gates, gates + n);
  c.M = M;
  c.dtype = dtype;
  *out = c.plan;
  g_plan_cache.insert(g_plan_cache.begin(), std::move(c));
  if (g_plan_cache.size() > 8) g_plan_cache.pop_back();
  return QSIM_OK;
}

// The gather wants most of the unified L1/shared array as L1 (the reuse
// cache of k1 lines): ask for the smallest carveout that still fits
// blocks_per_sm CTAs (4 KB sigma tables + 1 KB driver reserve each).
template <typename T, int U, int THREADS>
void launch_apply_sigma_u(int bps, unsigned blocks, const qsim::SigmaParams& sp,
                          const uint32_t* perm, uint64_t N, const T* k1, T* k2, cudaStream_t st) {
  const int pct = (bps * 5200 * 100 + 228 * 1024 - 1) / (228 * 1024);
  cudaFuncSetAttribute(qsim::k_apply_sigma<T, U, THREADS>,
                       cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
  qsim::k_apply_sigma<T, U, THREADS><<<blocks, THREADS, 0, st>>>(sp, perm, N, k1, k2);
}

// gathers in flight per thread, capped so the register budget of large CTAs
// holds them without spills (complex128 entries take four registers each)
template <typename T, int U>
void launch_apply_sigma_t(uint32_t threads, int bps, unsigned blocks, const qsim::SigmaParams& sp,
                          const uint32_t* perm, uint64_t N, const T* k1, T* k2, cudaStream_t st) {
  constexpr bool wide = sizeof(T) == 16;
  constexpr int U512 = wide && U > 16 ? 16 : U;
  constexpr int U1024 = wide ? (U > 8 ? 8 : U) : (U > 16 ? 16 : U);
  if (threads == 512) launch_apply_sigma_u<T, U512, 512>(bps, blocks, sp, perm, N, k1, k2, st);
  else if (threads == 1024) launch_apply_sigma_u<T, U1024, 1024>(bps, blocks, sp, perm, N, k1, k2, st);
  else launch_apply_sigma_u<T, U, 256>(bps, blocks, sp, perm, N, k1, k2, st);
}

template <typename T>
void launch_apply_sigma(uint32_t ilp, uint32_t threads, int bps, unsigned blocks,
                        const qsim::SigmaParams& sp, const uint32_t* perm, uint64_t N, const T* k1,
                        T* k2, cudaStream_t st) {
  if (ilp == 8) launch_apply_sigma_t<T, 8>(threads, bps, blocks, sp, perm, N, k1, k2, st);
  else if (ilp == 32) launch_apply_sigma_t<T, 32>(threads, bps, blocks, sp, perm, N, k1, k2, st);
  else launch_apply_sigma_t<T, 16>(threads, bps, blocks, sp, perm, N, k1, k2, st);
}


// Locality-keeping circuits (plan flag bit 1, re-checked on the gates given):
// the shared-memory staged kernel.  True if launched.
bool local_dispatch(const qsim_plan* plan, const qsim_gate* gates, int32_t n, const void* k1,
                    void* k2, uint32_t* perm_out, void* workspace, cudaStream_t st) {
  const int T = local_tile_bits(plan->dtype);
  if (!(plan->flags & 2u) || plan->M < T || moved_bits(gates, n) > T) return false;
  std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
  pack_gates(gates, n, false, *gl);
  std::string err;
  if (qsim::jit_local(gl->w, n, plan->M, elem_bytes(plan->dtype), T, k1, k2, perm_out, sm_count(),
                      st, err) != 0)
    return false;
  ++g_launches;
  g_last_kernel = "qsim_jit_local";
  return true;
}

// A natural-order plan still runs the NVRTC kernels (one pass, the walk in
// registers): identity sigma, chunks of up to
// 2^13 counters (all 8 warps of a CTA busy).
qsim_plan natural_view(const qsim_plan* plan) {
  qsim_plan p = *plan;
  for (int k = 0; k < 32; ++k) p.sigma[k] = (uint8_t)k;
  p.flags = 0;
  p.blocks_per_sm = 1;
  p.chunk_log2 = p.fused_chunk_log2 = (uint32_t)std::min(13, std::max(10, p.M - 7));
  return p;
}

int apply_planned_impl(const qsim_plan* plan, const uint32_t* perm, const void* k1, void* k2,
                       void* workspace, cudaStream_t st) {
  int rc = plan_validate(plan);
  if (rc) return rc;
  const int M = plan->M;
  const int e = elem_bytes(plan->dtype);
  if (!perm || !k1 || !k2 || !aligned16(perm) || !aligned16(k1) || !aligned16(k2))
    return QSIM_EINVAL;
  if (workspace && !aligned16(workspace)) return QSIM_EINVAL;
  const uint64_t N = 1ull << M;
  if (overlap(k1, N * e, k2, N * e) || overlap(perm, N * 4, k2, N * e)) return QSIM_EALIAS;
  const qsim_plan nat = natural_view(plan);
  const qsim_plan* pp = plan_natural(plan) ? &nat : plan;
  if (!plan_natural(plan) || M >= 13) {
    // NVRTC: the step kernel's traversal and batching, sources from perm
    const uint64_t nchunks = N >> pp->fused_chunk_log2;
    uint64_t blocks = (uint64_t)sm_count() * pp->blocks_per_sm;
    if (blocks > nchunks) blocks = nchunks;
    std::string err;
    if (qsim::jit_apply(M, pp->sigma, pp->fused_chunk_log2, e, perm, k1, k2, ticket_for(plan, workspace),
                        (int)blocks, jit_warps(pp), st, err) == 0) {
      ++g_launches;
      g_last_kernel = "qsim_jit_apply";
      return QSIM_OK;
    }
  }
  if (plan_natural(plan)) {
    g_last_kernel = "k_apply";
    return apply_impl(perm, 1ull << M, M, plan->dtype, k1, k2, st);
  }
  g_last_kernel = "k_apply_sigma";
  const qsim::SigmaParams sp = plan_params(plan, workspace);
  if ((rc = reset_ticket(workspace, st))) return rc;
  const uint64_t nchunks = N >> sp.chunk_log2;
  uint64_t blocks = (uint64_t)sm_count() * plan->blocks_per_sm;
  if (blocks > nchunks) blocks = nchunks;
  const uint32_t ilp = plan->ilp ? plan->ilp : 16u;
  const uint32_t thr = plan->cta_threads ? plan->cta_threads : 256u;
  if (plan->dtype == QSIM_C64)
    launch_apply_sigma<uint2>(ilp, thr, plan->blocks_per_sm, (unsigned)blocks, sp, perm, N,
                              static_cast<const uint2*>(k1), static_cast<uint2*>(k2), st);
  else
    launch_apply_sigma<uint4>(ilp, thr, plan->blocks_per_sm, (unsigned)blocks, sp, perm, N,
                              static_cast<const uint4*>(k1), static_cast<uint4*>(k2), st);
  QSIM_CHECK_LAUNCH("k_apply_sigma");
  return QSIM_OK;
}

template <int CAP, typename T>
int launch_fused_sigma(const qsim_plan* plan, const qsim_gate* gates, int32_t n, const T* k1, T* k2,
                       void* workspace, cudaStream_t st) {
  std::unique_ptr<qsim::GateList<CAP>> gl(new qsim::GateList<CAP>);
  pack_gates<CAP>(gates, n, true, *gl);
  const qsim::SigmaParams sp = plan_params(plan, workspace, true);
  int rc = reset_ticket(workspace, st);
  if (rc) return rc;
  const uint64_t N = 1ull << plan->M;
  const uint64_t nchunks = N >> sp.chunk_log2;
  uint64_t blocks = (uint64_t)sm_count() * plan->blocks_per_sm;
  if (blocks > nchunks) blocks = nchunks;
  const size_t smem = qsim::bs_smem_bytes((uint32_t)n);
  cudaFuncSetAttribute(qsim::k_fused_sigma<CAP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  // leave the rest of the unified array to L1 (reuse cache of k1 lines)
  const int pct = (int)(((smem + 1024) * plan->blocks_per_sm * 100 + 228 * 1024 - 1) / (228 * 1024));
  cudaFuncSetAttribute(qsim::k_fused_sigma<CAP, T>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       pct > 100 ? 100 : pct);
  qsim::k_fused_sigma<CAP, T><<<(unsigned)blocks, qsim::kBsThreads, smem, st>>>(*gl, sp, N, k1, k2);
  QSIM_CHECK_LAUNCH("k_fused_sigma");
  return QSIM_OK;
}

template <typename T>
int fused_planned_t(const qsim_plan* plan, const qsim_gate* gates, int32_t n, const T* k1, T* k2,
                    void* workspace, cudaStream_t st) {
  if (n <= 64) return launch_fused_sigma<64, T>(plan, gates, n, k1, k2, workspace, st);
  if (n <= 256) return launch_fused_sigma<256, T>(plan, gates, n, k1, k2, workspace, st);
  if (n <= 1024) return launch_fused_sigma<1024, T>(plan, gates, n, k1, k2, workspace, st);
  return launch_fused_sigma<qsim::kMaxGates, T>(plan, gates, n, k1, k2, workspace, st);
}

// Sigma-ordered fused kernel compiled for the circuit (qsim_jit.cu), or the
// shared-memory interpreter if NVRTC is unavailable.  perm_out != null also
// stores the map (one-pass map + gather).
int fused_sigma_dispatch(const qsim_plan* plan, const qsim_gate* gates, int32_t n, const void* k1,
                         void* k2, uint32_t* perm_out, void* workspace, cudaStream_t st,
                         bool* used_jit) {
  *used_jit = false;
  const int e = elem_bytes(plan->dtype);
  {  // workspace == nullptr: the kernel takes its chunks round-robin by CTA
    std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
    pack_gates(gates, n, false, *gl);
    std::string err;
    const uint64_t nchunks = (1ull << plan->M) >> plan->fused_chunk_log2;
    uint64_t blocks = (uint64_t)sm_count() * plan->blocks_per_sm;
    if (blocks > nchunks) blocks = nchunks;
    if (qsim::jit_fused(gl->w, n, plan->M, plan->sigma, plan->fused_chunk_log2, e, k1, k2, perm_out,
                        workspace, (int)blocks, jit_warps(plan), st, err) == 0) {
      ++g_launches;
      *used_jit = true;
      g_last_kernel = "qsim_jit_fused";
      return QSIM_OK;
    }
  }
  if (perm_out) return QSIM_EINVAL;  // caller handles the two-kernel fallback
  g_last_kernel = "k_fused_sigma";
  if (plan->dtype == QSIM_C64)
    return fused_planned_t<uint2>(plan, gates, n, static_cast<const uint2*>(k1),
                                  static_cast<uint2*>(k2), workspace, st);
  return fused_planned_t<uint4>(plan, gates, n, static_cast<const uint4*>(k1),
                                static_cast<uint4*>(k2), workspace, st);
}

int fused_planned_impl(const qsim_plan* plan, const qsim_gate* gates, int32_t n, const void* k1,
                       void* k2, void* workspace, cudaStream_t st) {
  int rc = plan_validate(plan);
  if (rc) return rc;
  const int M = plan->M;
  if ((rc = check_gates(gates, n, M))) return rc;
  {
    const int e = elem_bytes(plan->dtype);
    if (!k1 || !k2 || !aligned16(k1) || !aligned16(k2)) return QSIM_EINVAL;
    if (workspace && !aligned16(workspace)) return QSIM_EINVAL;
    if (overlap(k1, (1ull << M) * e, k2, (1ull << M) * e)) return QSIM_EALIAS;
  }
  if (local_dispatch(plan, gates, n, k1, k2, nullptr, workspace, st)) return QSIM_OK;
  if (plan_natural(plan)) {
    if (M >= 13) {
      const qsim_plan nat = natural_view(plan);
      bool jit = false;
      const int launches = g_launches;
      if (fused_sigma_dispatch(&nat, gates, n, k1, k2, nullptr, ticket_for(plan, workspace), st, &jit) ==
              QSIM_OK && jit)
        return QSIM_OK;
      g_launches = launches;
    }
    g_last_kernel = "k_fused_bitsliced";
    return fused_impl(gates, n, M, plan->dtype, 0, 1ull << M, k1, k2, QSIM_WALK_AUTO, st);
  }
  bool jit = false;
  return fused_sigma_dispatch(plan, gates, n, k1, k2, nullptr, workspace, st, &jit);
}

int map_gather_impl(const qsim_plan* plan, const qsim_gate* gates, int32_t n, uint32_t* perm,
                    const void* k1, void* k2, void* workspace, cudaStream_t st) {
  int rc = plan_validate(plan);
  if (rc) return rc;
  const int M = plan->M;
  if ((rc = check_gates(gates, n, M))) return rc;
  if (has_phase(gates, n)) {  // the stored map would drop the -1 rows
    std::snprintf(g_err, sizeof g_err, "phase gates: use qsim_build_map_signed");
    return QSIM_EINVAL;
  }
  const int e = elem_bytes(plan->dtype);
  if (!perm || !k1 || !k2 || !aligned16(perm) || !aligned16(k1) || !aligned16(k2))
    return QSIM_EINVAL;
  if (workspace && !aligned16(workspace)) return QSIM_EINVAL;
  const uint64_t N = 1ull << M;
  if (overlap(k1, N * e, k2, N * e) || overlap(perm, N * 4, k2, N * e) ||
      overlap(perm, N * 4, k1, N * e))
    return QSIM_EALIAS;
  if (local_dispatch(plan, gates, n, k1, k2, perm, workspace, st)) return QSIM_OK;
  if ((plan->flags & QSIM_PLAN_SPLIT) && !plan_natural(plan)) {
    // two kernels, each at its own best pattern: the planned gather with the
    // map recomputed in registers (k2 only), then the natural-order build
    // (perm written in coalesced runs instead of the gather's scattered
    // 64-128-byte runs, which cost one DRAM row activation each)
    bool jit = false;
    if ((rc = fused_sigma_dispatch(plan, gates, n, k1, k2, nullptr, workspace, st, &jit))) return rc;
    if ((rc = build_impl(gates, n, M, 0, N, perm, QSIM_WALK_AUTO, st))) return rc;
    g_last_kernel = jit ? "qsim_jit_fused + qsim_jit_build" : "k_fused_sigma + build";
    return QSIM_OK;
  }
  if (!plan_natural(plan) || M >= 13) {
    const qsim_plan nat = natural_view(plan);
    const qsim_plan* pp = plan_natural(plan) ? &nat : plan;
    bool jit = false;
    int launches = g_launches;
    rc = fused_sigma_dispatch(pp, gates, n, k1, k2, perm, ticket_for(plan, workspace), st, &jit);
    if (rc == QSIM_OK && jit) return QSIM_OK;
    g_launches = launches;
  }
  // two kernels: build (natural order, coalesced) then the planned gather
  rc = build_impl(gates, n, M, 0, N, perm, QSIM_WALK_AUTO, st);
  if (rc) return rc;
  const int32_t launches = g_launches;
  rc = apply_planned_impl(plan, perm, k1, k2, workspace, st);
  g_launches += launches;
  g_last_kernel = "build + apply";
  return rc;
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
  g_last_kernel = "";
  if (M < 1 || M > 32) return QSIM_ERANGE;
  // the whole output: planned internally (plan cached per circuit), the
  // NVRTC kernel in the plan's order -- the same bytes as every other path
  int rc = check_gates(gates, n_gates, M);
  if (rc == QSIM_OK && M >= 13 && elem_bytes(dtype) != 0 && qsim::jit_available()) {
    qsim_plan plan;
    if ((rc = cached_plan(gates, n_gates, M, dtype, &plan))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return fused_planned_impl(&plan, gates, n_gates, k1, k2, stream_ticket(st), st);
  }
  g_last_kernel = "k_fused_bitsliced";
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

int qsim_run_fused_kron(const qsim_gate* gates, int32_t n_gates, int32_t M, int32_t dtype,
                        const double* qubits, uint64_t start, uint64_t count, void* k2_out,
                        int32_t walk, void* stream) {
  g_launches = 0;
  g_last_kernel = "";
  return kron_impl(gates, n_gates, M, dtype, qubits, start, count, k2_out, walk,
                   static_cast<cudaStream_t>(stream));
}

int qsim_plan_create(const qsim_gate* gates, int32_t n, int32_t M, int32_t dtype,
                     qsim_plan* plan) {
  g_launches = 0;
  int rc = check_gates(gates, n, M);
  if (rc) return rc;
  if (!plan || elem_bytes(dtype) == 0) return QSIM_EINVAL;
  return plan_fill(gates, n, M, dtype, plan);
}

int qsim_apply_map_planned(const qsim_plan* plan, const uint32_t* perm, const void* k1, void* k2,
                           void* workspace, void* stream) {
  g_launches = 0;
  g_last_kernel = "";
  return apply_planned_impl(plan, perm, k1, k2, workspace, static_cast<cudaStream_t>(stream));
}

int qsim_run_fused_planned(const qsim_plan* plan, const qsim_gate* gates, int32_t n_gates,
                           const void* k1, void* k2, void* workspace, void* stream) {
  g_launches = 0;
  g_last_kernel = "";
  return fused_planned_impl(plan, gates, n_gates, k1, k2, workspace,
                            static_cast<cudaStream_t>(stream));
}

int qsim_build_map_signed(const qsim_gate* gates, int32_t n_gates, int32_t M, uint64_t start,
                          uint64_t count, uint32_t* perm, uint32_t* signs, void* stream) {
  g_launches = 0;
  if (M < 1 || M > 32) return QSIM_ERANGE;
  return build_signed_impl(gates, n_gates, M, start, count, perm, signs,
                           static_cast<cudaStream_t>(stream));
}

int qsim_apply_map_signed(const uint32_t* perm, const uint32_t* signs, uint64_t count, int32_t M,
                          int32_t dtype, const void* k1, void* k2, void* stream) {
  g_launches = 0;
  return apply_signed_impl(perm, signs, count, M, dtype, k1, k2, static_cast<cudaStream_t>(stream));
}

int qsim_map_gather_planned(const qsim_plan* plan, const qsim_gate* gates, int32_t n_gates,
                            uint32_t* perm, const void* k1, void* k2, void* workspace,
                            void* stream) {
  g_launches = 0;
  g_last_kernel = "";
  return map_gather_impl(plan, gates, n_gates, perm, k1, k2, workspace,
                         static_cast<cudaStream_t>(stream));
}

int qsim_run_host(const qsim_gate* gates, int32_t n_gates, int32_t M, int32_t dtype, int32_t mode,
                  const void* k1_host, void* k2_host, void* k1_dev, void* k2_dev,
                  uint32_t* perm_dev, void* workspace, void* stream) {
  g_launches = 0;
  int rc = check_gates(gates, n_gates, M);
  if (rc) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0 || (mode != 0 && mode != 1)) return QSIM_EINVAL;
  if (!k1_host || !k2_host || !k1_dev || !k2_dev) return QSIM_EINVAL;
  if (mode == 0 && !perm_dev) return QSIM_EINVAL;
  if (mode == 0 && has_phase(gates, n_gates)) return QSIM_EINVAL;  // map + gather stores the map
  const uint64_t N = 1ull << M, bytes = N * e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // validate the compute step before enqueuing anything
  if (!aligned16(k1_dev) || !aligned16(k2_dev) || (mode == 0 && !aligned16(perm_dev)) ||
      (workspace && !aligned16(workspace)))
    return QSIM_EINVAL;
  if (overlap(k1_dev, bytes, k2_dev, bytes) ||
      (mode == 0 && (overlap(perm_dev, N * 4, k2_dev, bytes) ||
                     overlap(perm_dev, N * 4, k1_dev, bytes))))
    return QSIM_EALIAS;
  qsim_plan plan;
  if ((rc = cached_plan(gates, n_gates, M, dtype, &plan))) return rc;
  cudaError_t ce = cudaMemcpyAsync(k1_dev, k1_host, bytes, cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "H2D k1");
  int launches = 0;
  if (mode == 0) {
    rc = map_gather_impl(&plan, gates, n_gates, perm_dev, k1_dev, k2_dev, workspace, st);
  } else {
    rc = fused_planned_impl(&plan, gates, n_gates, k1_dev, k2_dev, workspace, st);
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

int qsim_run_host_batch(const qsim_gate* gates, int32_t n_gates, int32_t M, int32_t dtype,
                        int32_t mode, int32_t nsteps, const void* const* k1_hosts,
                        void* const* k2_hosts, void* k1_dev0, void* k1_dev1, void* k2_dev0,
                        void* k2_dev1, uint32_t* perm_dev, void* workspace) {
  g_launches = 0;
  int rc = check_gates(gates, n_gates, M);
  if (rc) return rc;
  const int e = elem_bytes(dtype);
  if (e == 0 || (mode != 0 && mode != 1) || nsteps < 0) return QSIM_EINVAL;
  if (nsteps > 0 && (!k1_hosts || !k2_hosts)) return QSIM_EINVAL;
  for (int32_t i = 0; i < nsteps; ++i)
    if (!k1_hosts[i] || !k2_hosts[i]) return QSIM_EINVAL;
  void* k1d[2] = {k1_dev0, k1_dev1};
  void* k2d[2] = {k2_dev0, k2_dev1};
  const uint64_t N = 1ull << M, bytes = N * e;
  for (int b = 0; b < 2; ++b)
    if (!k1d[b] || !k2d[b] || !aligned16(k1d[b]) || !aligned16(k2d[b])) return QSIM_EINVAL;
  if (mode == 0 && (!perm_dev || !aligned16(perm_dev))) return QSIM_EINVAL;
  if (mode == 0 && has_phase(gates, n_gates)) return QSIM_EINVAL;
  if (workspace && !aligned16(workspace)) return QSIM_EINVAL;
  const void* bufs[5] = {k1d[0], k1d[1], k2d[0], k2d[1], perm_dev};
  const uint64_t sz[5] = {bytes, bytes, bytes, bytes, mode == 0 ? N * 4 : 0};
  for (int a = 0; a < 5; ++a)
    for (int b = a + 1; b < 5; ++b)
      if (overlap(bufs[a], sz[a], bufs[b], sz[b])) return QSIM_EALIAS;
  if (nsteps == 0) return QSIM_OK;
  qsim_plan plan;
  if ((rc = cached_plan(gates, n_gates, M, dtype, &plan))) return rc;
  // three streams: copies in, compute, copies out; step i uses buffer i & 1
  cudaStream_t sin = nullptr, scmp = nullptr, sout = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_cmp[2] = {nullptr, nullptr},
              ev_out[2] = {nullptr, nullptr};
  cudaError_t ce = cudaSuccess;
  auto cleanup = [&]() {
    for (int b = 0; b < 2; ++b) {
      if (ev_in[b]) cudaEventDestroy(ev_in[b]);
      if (ev_cmp[b]) cudaEventDestroy(ev_cmp[b]);
      if (ev_out[b]) cudaEventDestroy(ev_out[b]);
    }
    if (sin) cudaStreamDestroy(sin);
    if (scmp) cudaStreamDestroy(scmp);
    if (sout) cudaStreamDestroy(sout);
  };
  if ((ce = cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking)) != cudaSuccess ||
      (ce = cudaStreamCreateWithFlags(&scmp, cudaStreamNonBlocking)) != cudaSuccess ||
      (ce = cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking)) != cudaSuccess) {
    cleanup();
    return cuda_fail(ce, "stream create");
  }
  for (int b = 0; b < 2 && ce == cudaSuccess; ++b) {
    if ((ce = cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming)) != cudaSuccess) break;
    if ((ce = cudaEventCreateWithFlags(&ev_cmp[b], cudaEventDisableTiming)) != cudaSuccess) break;
    ce = cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming);
  }
  if (ce != cudaSuccess) {
    cleanup();
    return cuda_fail(ce, "event create");
  }
  // Iteration i copies step i in and step i-1 out, interleaved in 256 MB
  // chunks on the two copy streams (PCIe is full duplex: ~50 GB/s each way
  // together, 55 alone), then enqueues step i's compute.
  const uint64_t chunk = 256ull << 20;
  int launches = 0;
  for (int32_t i = 0; i <= nsteps && rc == QSIM_OK; ++i) {
    const int b = i & 1, bp = (i - 1) & 1;
    const bool in = i < nsteps, out = i >= 1;
    // k1[b] is free once step i-2's compute has read it; k2[bp] is ready after step i-1
    if (in && i >= 2 && (ce = cudaStreamWaitEvent(sin, ev_cmp[b], 0)) != cudaSuccess) break;
    if (out && (ce = cudaStreamWaitEvent(sout, ev_cmp[bp], 0)) != cudaSuccess) break;
    for (uint64_t o = 0; o < bytes && ce == cudaSuccess; o += chunk) {
      const uint64_t c = std::min(chunk, bytes - o);
      if (in)
        ce = cudaMemcpyAsync(static_cast<char*>(k1d[b]) + o,
                             static_cast<const char*>(k1_hosts[i]) + o, c, cudaMemcpyHostToDevice,
                             sin);
      if (out && ce == cudaSuccess)
        ce = cudaMemcpyAsync(static_cast<char*>(k2_hosts[i - 1]) + o,
                             static_cast<const char*>(k2d[bp]) + o, c, cudaMemcpyDeviceToHost,
                             sout);
    }
    if (ce != cudaSuccess) break;
    if (out && (ce = cudaEventRecord(ev_out[bp], sout)) != cudaSuccess) break;
    if (!in) break;
    if ((ce = cudaEventRecord(ev_in[b], sin)) != cudaSuccess) break;
    // compute: its input is in, and k2[b] has been copied out by step i-2
    if ((ce = cudaStreamWaitEvent(scmp, ev_in[b], 0)) != cudaSuccess) break;
    if (i >= 2 && (ce = cudaStreamWaitEvent(scmp, ev_out[b], 0)) != cudaSuccess) break;
    rc = mode == 0 ? map_gather_impl(&plan, gates, n_gates, perm_dev, k1d[b], k2d[b], workspace, scmp)
                   : fused_planned_impl(&plan, gates, n_gates, k1d[b], k2d[b], workspace, scmp);
    launches += g_launches;
    if (rc) break;
    if ((ce = cudaEventRecord(ev_cmp[b], scmp)) != cudaSuccess) break;
  }
  cudaError_t ce2 = cudaStreamSynchronize(sin);
  if (ce2 == cudaSuccess) ce2 = cudaStreamSynchronize(scmp);
  if (ce2 == cudaSuccess) ce2 = cudaStreamSynchronize(sout);
  cleanup();
  if (rc) return rc;
  if (ce != cudaSuccess) return cuda_fail(ce, "qsim_run_host_batch");
  if (ce2 != cudaSuccess) return cuda_fail(ce2, "qsim_run_host_batch sync");
  g_launches = launches;
  return QSIM_OK;
}

// qsim_plan_tune stage 4: rounds of screening every exchange of two counter positions
constexpr int kTuneSwapRounds = 2;
// stage 5: rounds of exchanges of a compiled position with any later one
constexpr int kTuneCompiledRounds = 3;

int qsim_plan_tune(qsim_plan* plan, const qsim_gate* gates, int32_t n_gates, uint32_t* perm,
                   const void* k1, void* k2, void* workspace, void* stream, int32_t* chosen) {
  return qsim_plan_tune_ex(plan, gates, n_gates, perm, k1, k2, workspace, stream, QSIM_TUNE_PATIENT,
                           chosen);
}

int qsim_plan_tune_ex(qsim_plan* plan, const qsim_gate* gates, int32_t n_gates, uint32_t* perm,
                      const void* k1, void* k2, void* workspace, void* stream, int32_t effort,
                      int32_t* chosen) {
  g_launches = 0;
  if (!plan || !workspace || !aligned16(workspace)) return QSIM_EINVAL;
  // QSIM_TUNE_APPLY: the trials time qsim_apply_map_planned on the map in perm
  // (built once here) instead of the map + gather step
  const bool for_apply = (effort & QSIM_TUNE_APPLY) != 0;
  effort &= ~QSIM_TUNE_APPLY;
  if (effort != QSIM_TUNE_MEASURE && effort != QSIM_TUNE_PATIENT) return QSIM_EINVAL;
  int rc = plan_validate(plan);
  if (rc) return rc;
  if ((rc = check_gates(gates, n_gates, plan->M))) return rc;
  if (has_phase(gates, n_gates)) return QSIM_EINVAL;  // tunes the map + gather step
  {  // the buffers every trial call uses (validated once, before anything runs)
    const uint64_t N = 1ull << plan->M;
    const int e = elem_bytes(plan->dtype);
    if (!perm || !k1 || !k2 || !aligned16(perm) || !aligned16(k1) || !aligned16(k2))
      return QSIM_EINVAL;
    if (overlap(k1, N * e, k2, N * e) || overlap(perm, N * 4, k2, N * e) ||
        overlap(perm, N * 4, k1, N * e))
      return QSIM_EALIAS;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (for_apply && (rc = build_impl(gates, n_gates, plan->M, 0, 1ull << plan->M, perm, QSIM_WALK_AUTO, st)))
    return rc;
  // candidates: the default rule, the full cover, each with lanes on output bits 0..4,
  // and smaller full covers
  const PlanOpts base;
  std::vector<PlanOpts> opts;
  for (int fixed = 0; fixed < 2; ++fixed)
    for (int run = 0; run < 2; ++run) {
      PlanOpts o = base;
      o.fixed = fixed != 0;
      o.lane_run = run != 0;
      opts.push_back(o);
    }
  for (int T = base.cover_bits - 2; T < base.cover_bits; ++T) {
    PlanOpts o = base;
    o.cover_bits = T;
    o.fixed = true;
    opts.push_back(o);
  }

  std::vector<qsim_plan> cands;
  std::vector<int> idx;
  for (size_t i = 0; i < opts.size(); ++i) {
    qsim_plan p;
    if ((rc = plan_fill(gates, n_gates, plan->M, plan->dtype, &p, opts[i]))) return rc;
    p.chunk_log2 = plan->chunk_log2;
    p.fused_chunk_log2 = plan->fused_chunk_log2;
    p.blocks_per_sm = plan->blocks_per_sm;
    bool dup = false;
    for (const qsim_plan& c : cands)
      dup = dup || (std::memcmp(c.sigma, p.sigma, 32) == 0 && c.flags == p.flags);
    if (!dup) {
      cands.push_back(p);
      idx.push_back((int)i);
    }
  }
  // each sigma variant also as the two-kernel step (planned gather, then the
  // natural-order build): cfg5 14.9 + 2.7 ms against 18.0 ms for one kernel
  // storing perm in plan order (profiles/r02_concurrent_build.txt)
  for (size_t i = 0, nc = for_apply ? 0 : cands.size(); i < nc; ++i)
    if (!plan_natural(&cands[i]) && !(cands[i].flags & 2u)) {
      qsim_plan p = cands[i];
      p.flags |= QSIM_PLAN_SPLIT;
      cands.push_back(p);
      idx.push_back(idx[i] + 8);
    }
  cudaEvent_t a = nullptr, b = nullptr;
  cudaError_t ce;
  if ((ce = cudaEventCreate(&a)) != cudaSuccess || (ce = cudaEventCreate(&b)) != cudaSuccess) {
    if (a) cudaEventDestroy(a);
    return cuda_fail(ce, "event create");
  }
  // best of `reps` timed map + gather calls with plan p (one untimed call
  // first when `warm`: it compiles the kernel)
  auto trial = [&](const qsim_plan& p) -> int {
    return for_apply ? apply_planned_impl(&p, perm, k1, k2, workspace, st)
                     : map_gather_impl(&p, gates, n_gates, perm, k1, k2, workspace, st);
  };
  auto time_plan = [&](const qsim_plan& p, bool warm, int reps) -> float {
    if (warm && (rc = trial(p))) return 1e30f;
    float t_best = 1e30f;
    for (int r = 0; r < reps && rc == QSIM_OK; ++r) {
      cudaEventRecord(a, st);
      rc = trial(p);
      cudaEventRecord(b, st);
      if ((ce = cudaEventSynchronize(b)) != cudaSuccess) {
        rc = cuda_fail(ce, "tune sync");
        break;
      }
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, a, b);
      t_best = std::min(t_best, ms);
    }
    return rc == QSIM_OK ? t_best : 1e30f;
  };
  float best = 1e30f;
  int best_i = -1;
  for (size_t i = 0; i < cands.size() && rc == QSIM_OK; ++i) {
    const float t = time_plan(cands[i], true, 2);
    if (rc == QSIM_OK && t < best) {
      best = t;
      best_i = (int)i;
    }
  }
  if (rc != QSIM_OK || best_i < 0) {  // a trial failed: nothing was kept
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return rc != QSIM_OK ? rc : QSIM_EINVAL;
  }
  // second stage: the chunk size of the kept order (2^14 / 2^16 next to 2^15)
  qsim_plan kept = cands[best_i];
  const uint32_t c0 = kept.fused_chunk_log2;
  for (int d = -1; d <= 1 && rc == QSIM_OK; d += 2) {
    const int cl = (int)c0 + d;
    if (cl < 10 || cl > kept.M || ((1ull << kept.M) >> cl) < (uint64_t)sm_count()) continue;
    qsim_plan p = kept;
    p.chunk_log2 = p.fused_chunk_log2 = (uint32_t)cl;
    const float t = time_plan(p, false, 2);
    if (rc == QSIM_OK && t < best * 0.99f) {  // only a clear win moves it
      best = t;
      cands[best_i] = p;
    }
  }
  // third stage: the order of the counter bits above the cover (runtime
  // kernel parameter, no recompiles).  The plan orders them for the k1 reads
  // (a line's readers close in time); moving an output bit down next to the
  // cover changes which k2 / perm lines share a chunk front (their DRAM rows
  // on write-back) and which k1 lines are read together.  Best-improvement
  // rounds: every tail bit tried at each of the 10 positions just above the
  // cover (screened with one timed call), the four best re-timed (best of
  // three) and the best kept on a >= 0.5 % win; up to 3 rounds.  The gains
  // depend on the data in the buffers (power: sw_power_cap), which is why the
  // search runs on the caller's buffers.  cfg5: output bit 4 moves from
  // counter bit 21 to 15, 19.85 -> 19.3 ms with the bench's Gaussian state;
  // with an index-valued state output bit 28 next to the cover gains 1.8 %
  // more (profiles/r02_sigma_tail_moves.txt, r02_tail_search.txt,
  // r02_sigma_ab.txt).
  qsim_plan cur = cands[best_i];
  const int from = std::max(10, (int)cur.tile_log2);
  if (!(cur.flags & 1u) && cur.M >= from + 4) {
    const bool trace = std::getenv("QSIM_TUNE_TRACE") != nullptr;  // diagnostics (stderr)
    float cur_t = time_plan(cur, false, 3);
    // Stages 3-5 share one step: screen every candidate order with one timed
    // call (the GPU kept busy first, so no screen profits from an idle,
    // unthrottled start -- the bench state runs into sw_power_cap), then
    // re-time the four best against the current order interleaved (cur,
    // cand, cur, cand, ...: best of 3 each, so clock drift cancels) and keep
    // the best ratio when it is a >= 0.5 % win.  Returns true if cur moved.
    // (compiled: a candidate's first call may load its kernel -- it is warmed untimed)
    auto step = [&](const std::vector<qsim_plan>& cand_plans, const char* stage, bool compiled) -> bool {
      time_plan(cur, false, 2);
      std::vector<std::pair<float, size_t>> screened;
      for (size_t c = 0; c < cand_plans.size() && rc == QSIM_OK; ++c) {
        const float t = time_plan(cand_plans[c], compiled, 1);
        if (rc == QSIM_OK) screened.push_back({t, c});
      }
      if (rc != QSIM_OK || screened.empty()) return false;
      const size_t top = std::min<size_t>(4, screened.size());
      std::partial_sort(screened.begin(), screened.begin() + top, screened.end());
      float best_ratio = 1.0f, best_t = cur_t;
      size_t best_c = SIZE_MAX;
      for (size_t c = 0; c < top && rc == QSIM_OK; ++c) {
        float tc = 1e30f, tx = 1e30f;
        for (int r = 0; r < 3 && rc == QSIM_OK; ++r) {
          tc = std::min(tc, time_plan(cur, false, 1));
          tx = std::min(tx, time_plan(cand_plans[screened[c].second], false, 1));
        }
        if (trace)
          std::fprintf(stderr, "[qsim_plan_tune] %s: screened %.3f, re-timed %.3f vs current %.3f\n", stage,
                       screened[c].first, tx, tc);
        if (rc == QSIM_OK && tx / tc < best_ratio) {
          best_ratio = tx / tc;
          best_t = tx;
          best_c = screened[c].second;
        }
      }
      if (rc != QSIM_OK || best_c == SIZE_MAX || !(best_ratio < 0.995f)) return false;
      cur = cand_plans[best_c];
      cur_t = best_t;
      return true;
    };
    // third stage: the order of the counter bits above the cover (runtime
    // kernel parameter, no recompiles).  The plan orders them for the k1 reads
    // (a line's readers close in time); moving an output bit down next to the
    // cover changes which k2 / perm lines share a chunk front (their DRAM rows
    // on write-back) and which k1 lines are read together: every tail bit
    // tried at each of the 10 positions just above the cover; up to 3 rounds.
    // The gains depend on the data in the buffers (power: sw_power_cap),
    // which is why the search runs on the caller's buffers.  cfg5: output bit
    // 4 moves from counter bit 21 to 15, 19.85 -> 19.3 ms with the bench's
    // Gaussian state (profiles/r02_sigma_tail_moves.txt, r02_tail_search.txt,
    // r02_sigma_ab.txt).
    for (int round = 0; round < 3 && rc == QSIM_OK; ++round) {
      std::vector<qsim_plan> moves;
      for (int at = from; at < cur.M; ++at)
        for (int pos = from; pos < std::min(cur.M, from + 10); ++pos) {
          if (pos == at) continue;
          qsim_plan p = cur;
          uint8_t rest[32];
          int m = 0;
          for (int k = from; k < cur.M; ++k)
            if (k != at) rest[m++] = cur.sigma[k];
          for (int k = from, r = 0; k < cur.M; ++k) p.sigma[k] = k == pos ? cur.sigma[at] : rest[r++];
          moves.push_back(p);
        }
      if (!step(moves, "stage 3", false)) break;
    }
    // fourth stage: exchanges of any two counter positions >= 10 (this also
    // trades the CTA's warp-level cover bits 10..12 against tail bits); up to
    // 2 rounds.  cfg5: a random-swap hill climb found 19.11 -> 18.81 ms
    // (tools/exp/tail_climb.py, profiles/r02_tail_climb.txt)
    auto swap_rounds = [&](int rounds) {
      for (int round = 0; round < rounds && rc == QSIM_OK; ++round) {
        std::vector<qsim_plan> swaps;
        for (int i = 10; i < cur.M; ++i)
          for (int j = i + 1; j < cur.M; ++j) {
            qsim_plan p = cur;
            std::swap(p.sigma[i], p.sigma[j]);
            swaps.push_back(p);
          }
        if (!step(swaps, "stage 4", false)) break;
      }
    };
    if (effort == QSIM_TUNE_PATIENT) swap_rounds(kTuneSwapRounds);
    // fifth stage: exchanges that move a compiled position (counter bits
    // plan_keep_bits..9: lanes and in-thread entries; each order is a new
    // NVRTC kernel, a round's kernels compiled at once on the host's cores)
    // with any later position; each kept move is followed by one more round
    // of the fourth stage; up to 3 rounds.  cfg5: lanes on output bit 11
    // instead of 3 (output bit 3 in-thread) 18.91 -> 18.35 ms, then output
    // bit 3 to the warp bits 18.20 -> 17.99 ms (tools/exp/compiled_swaps.py,
    // profiles/r02_compiled_swaps.txt)
    std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
    pack_gates(gates, n_gates, false, *gl);
    const unsigned hw = std::thread::hardware_concurrency();
    for (int round = 0; effort == QSIM_TUNE_PATIENT && round < kTuneCompiledRounds && rc == QSIM_OK;
         ++round) {
      std::vector<qsim_plan> cand_plans;
      const int keep = plan_keep_bits(cur.dtype);
      for (int i = keep; i < 10 && i < cur.M; ++i)
        for (int j = i + 1; j < cur.M; ++j) {
          qsim_plan p = cur;
          std::swap(p.sigma[i], p.sigma[j]);
          cand_plans.push_back(p);
        }
      std::vector<uint8_t> sg(32 * cand_plans.size());
      for (size_t c = 0; c < cand_plans.size(); ++c) std::memcpy(&sg[32 * c], cand_plans[c].sigma, 32);
      qsim::jit_fused_prepare(gl->w, n_gates, cur.M, sg.data(), (int)cand_plans.size(), elem_bytes(cur.dtype),
                              jit_warps(&cur), hw ? (int)std::min(hw, 32u) : 8, for_apply);
      if (!step(cand_plans, "stage 5", true)) break;
      swap_rounds(1);
    }
    // sixth stage: the chunk size, 2 CTAs per SM and 16-warp CTAs, for the
    // order kept (stage 2 chose the chunk for the stage-1 order; cfg5 keeps
    // 2^15 counters, 1 CTA of 8 warps: 16 warps 18.7 vs 17.75 ms,
    // profiles/r02_cta16.txt)
    {
      std::vector<qsim_plan> launch_cands;
      for (int d = -1; d <= 1; d += 2) {
        const int cl = (int)cur.fused_chunk_log2 + d;
        if (cl < 10 || cl > cur.M || ((1ull << cur.M) >> cl) < (uint64_t)sm_count()) continue;
        qsim_plan p = cur;
        p.chunk_log2 = p.fused_chunk_log2 = (uint32_t)cl;
        launch_cands.push_back(p);
      }
      if (cur.blocks_per_sm == 1) {
        qsim_plan p = cur;
        p.blocks_per_sm = 2;
        launch_cands.push_back(p);
      }
      if (cur.cta_threads == 256) {  // 16 warps per CTA: a round covers counter bits 0..13
        qsim_plan p = cur;
        p.cta_threads = 512;
        launch_cands.push_back(p);
      }
      if (effort == QSIM_TUNE_PATIENT && rc == QSIM_OK && !launch_cands.empty())
        step(launch_cands, "stage 6", true);
    }
    best = std::min(best, cur_t);
    if (rc == QSIM_OK) cands[best_i] = cur;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (rc) return rc;
  *plan = cands[best_i];
  if (chosen) *chosen = idx[best_i];
  g_launches = 0;
  return QSIM_OK;
}

struct qsim_graph {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  int32_t launches;
};

int qsim_graph_create(const qsim_plan* plan, const qsim_gate* gates, int32_t n_gates, int32_t call,
                      uint32_t* perm, const void* k1, void* k2, void* workspace, int32_t reps,
                      qsim_graph** out) {
  g_launches = 0;
  if (!out || reps < 1 || reps > 1024 || call < 0 || call > 2) return QSIM_EINVAL;
  *out = nullptr;
  auto step = [&](cudaStream_t st) {
    return call == 0   ? map_gather_impl(plan, gates, n_gates, perm, k1, k2, workspace, st)
           : call == 1 ? fused_planned_impl(plan, gates, n_gates, k1, k2, workspace, st)
                       : apply_planned_impl(plan, perm, k1, k2, workspace, st);
  };
  cudaStream_t st = nullptr;
  cudaError_t ce = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (ce != cudaSuccess) return cuda_fail(ce, "stream create");
  // one uncaptured step: validates, NVRTC-compiles and loads the kernels
  int rc = step(st);
  if (rc == QSIM_OK && (ce = cudaStreamSynchronize(st)) != cudaSuccess) rc = cuda_fail(ce, "warm-up");
  cudaGraph_t graph = nullptr;
  int32_t launches = 0;
  if (rc == QSIM_OK) {
    if ((ce = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) {
      rc = cuda_fail(ce, "begin capture");
    } else {
      for (int32_t r = 0; r < reps && rc == QSIM_OK; ++r) {
        rc = step(st);
        launches += g_launches;
      }
      ce = cudaStreamEndCapture(st, &graph);
      if (rc == QSIM_OK && ce != cudaSuccess) rc = cuda_fail(ce, "end capture");
    }
  }
  cudaGraphExec_t exec = nullptr;
  if (rc == QSIM_OK && (ce = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess)
    rc = cuda_fail(ce, "graph instantiate");
  cudaStreamDestroy(st);
  if (rc != QSIM_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  *out = new qsim_graph{graph, exec, launches};
  g_launches = 0;
  return QSIM_OK;
}

int qsim_graph_launch(qsim_graph* g, void* stream) {
  g_launches = 0;
  if (!g) return QSIM_EINVAL;
  cudaError_t ce = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream));
  if (ce != cudaSuccess) return cuda_fail(ce, "graph launch");
  g_launches = g->launches;
  return QSIM_OK;
}

int qsim_graph_destroy(qsim_graph* g) {
  g_launches = 0;
  if (!g) return QSIM_OK;
  cudaError_t e1 = cudaGraphExecDestroy(g->exec), e2 = cudaGraphDestroy(g->graph);
  delete g;
  if (e1 != cudaSuccess) return cuda_fail(e1, "graph exec destroy");
  if (e2 != cudaSuccess) return cuda_fail(e2, "graph destroy");
  return QSIM_OK;
}

int32_t qsim_last_launch_count(void) { return g_launches; }

const char* qsim_last_kernel(void) { return g_last_kernel; }

const char* qsim_strerror(int32_t code) {
  switch (code) {
    case QSIM_OK: return "ok";
    case QSIM_EINVAL: return "invalid argument (null/misaligned pointer, bad dtype/mode/kind/plan)";
    case QSIM_ERANGE: return "M outside [1, 32] or range outside [0, 2^M)";
    case QSIM_EBIT: return "gate bit out of range, target among controls, or duplicate control";
    case QSIM_ECAP: return "gate count outside [0, QSIM_MAX_GATES]";
    case QSIM_EALIAS: return "device buffers overlap";
    case QSIM_ECUDA: return "CUDA call failed (see qsim_last_error)";
    default: return "unknown qsim status";
  }
}

const char* qsim_last_error(void) { return g_err; }

const char* qsim_jit_status(void) { return qsim::jit_status(); }

double qsim_jit_last_compile_ms(void) { return qsim::jit_last_compile_ms(); }

int qsim_jit_check_compile_planned(const qsim_plan* plan, const qsim_gate* gates,
                                   int32_t n_gates) {
  g_launches = 0;
  int rc = plan_validate(plan);
  if (rc) return rc;
  if ((rc = check_gates(gates, n_gates, plan->M))) return rc;
  std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
  pack_gates(gates, n_gates, false, *gl);
  std::string err;
  if (qsim::jit_check_compile_fused(gl->w, n_gates, plan->M, plan->sigma, elem_bytes(plan->dtype),
                                    err) != 0) {
    std::snprintf(g_err, sizeof g_err, "jit: %s", err.c_str());
    return QSIM_ECUDA;
  }
  if (qsim::jit_check_compile_apply(plan->M, plan->sigma, elem_bytes(plan->dtype), err) != 0) {
    std::snprintf(g_err, sizeof g_err, "jit (apply): %s", err.c_str());
    return QSIM_ECUDA;
  }
  if ((plan->flags & 2u) && qsim::jit_check_compile_local(gl->w, n_gates, plan->M,
                                                          elem_bytes(plan->dtype),
                                                          local_tile_bits(plan->dtype), err) != 0) {
    std::snprintf(g_err, sizeof g_err, "jit (local tiles): %s", err.c_str());
    return QSIM_ECUDA;
  }
  return QSIM_OK;
}

int qsim_jit_check_compile_kron(const qsim_gate* gates, int32_t n_gates, int32_t M,
                                int32_t dtype) {
  g_launches = 0;
  int rc = check_gates_kron(gates, n_gates, M);
  if (rc) return rc;
  if (elem_bytes(dtype) == 0) return QSIM_EINVAL;
  std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
  pack_gates(gates, n_gates, false, *gl);
  std::string err;
  uint32_t gb = 0, ng = 0;
  kron_groups(M, elem_bytes(dtype), &gb, &ng);
  KronLayout ly;  // the layout of a call over all 2^M outputs
  kron_layout(gates, n_gates, M, (int)gb, (int)ng, 0, 1ull << M, true, &ly);
  if (qsim::jit_check_compile_kron(gl->w, n_gates, M, elem_bytes(dtype), (int)gb, (int)ng, ly.pos,
                                   ly.J, ly.L, ly.nv, err) != 0) {
    std::snprintf(g_err, sizeof g_err, "jit: %s", err.c_str());
    return QSIM_ECUDA;
  }
  return QSIM_OK;
}

int qsim_jit_check_compile(const qsim_gate* gates, int32_t n_gates, int32_t M) {
  g_launches = 0;
  int rc = check_gates(gates, n_gates, M);
  if (rc) return rc;
  std::unique_ptr<qsim::GateList<qsim::kMaxGates>> gl(new qsim::GateList<qsim::kMaxGates>);
  pack_gates(gates, n_gates, false, *gl);
  std::string err;
  ThreadBits tb;  // the in-thread bits of a call over all 2^M outputs (as build_impl)
  const char* bt = std::getenv("QSIM_BUILD_THREAD_BITS");
  thread_bits(gates, n_gates, M, 0, (bt && bt[0] == '0') ? 0 : 1ull << M, kBuildMaxV, true, &tb);
  if (qsim::jit_check_compile(gl->w, n_gates, M, tb.J, tb.L, tb.V, err) != 0) {
    std::snprintf(g_err, sizeof g_err, "jit: %s", err.c_str());
    return QSIM_ECUDA;
  }
  return QSIM_OK;
}

int32_t qsim_abi_version(void) { return 7; }

}  // extern "C"
