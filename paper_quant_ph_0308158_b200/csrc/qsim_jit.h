// qsim_jit.h -- run-time specialised walk kernels (internal to libqsim.so).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace qsim {
bool jit_available();
const char* jit_status();
double jit_last_compile_ms();
// NVRTC-compile the build kernel for this gate list without loading it
// (works without a GPU); 0 on success.
int jit_check_compile(const uint32_t* words, int n, int M, const uint8_t* J, int L, uint64_t V,
                      std::string& err);
// Build perm for outputs [start, start+count) with a kernel compiled for this
// exact gate list (per-lane word format).  Returns 0, or -1 with err set (the
// caller then uses the interpreter kernel).
// In-thread bits (qsim_api.cu thread_bits): J = output bits walked inside a
// thread, tiles fill aligned blocks of 2^L outputs, V != 0 enables the fast
// path (address bits outside V constant in a thread).
int jit_build(const uint32_t* words, int n, int M, const uint8_t* J, int L, uint64_t V,
              uint64_t start, uint64_t count, uint32_t* perm_out, int sms, cudaStream_t st,
              std::string& err);
// Sigma-ordered fused walk + gather over all 2^M outputs with a kernel
// compiled for (circuit, sigma[0..9], element size, warps per CTA: 8 or 16,
// tiles of 1024 counters striding by it); sigma[10..] is a kernel
// parameter.  If perm_out != null the map is stored as well (one-pass map +
// gather).  ticket: device scratch (reset on st).  Returns 0 or -1 with err.
int jit_fused(const uint32_t* words, int n, int M, const uint8_t* sigma, uint32_t chunk_log2,
              int elem, const void* k1, void* k2, uint32_t* perm_out, void* ticket, int blocks,
              int warps, cudaStream_t st, std::string& err);
// Compile (NVRTC, on up to `threads` host threads at once) and cache the fused
// kernels of `count` orders (32 bytes each, sigmas[32 * i ..]) that are not
// cached yet, so that later jit_fused calls find them.  Returns the number
// compiled, or -1 if NVRTC is unavailable.
int jit_fused_prepare(const uint32_t* words, int n, int M, const uint8_t* sigmas, int count, int elem,
                      int warps, int threads, bool apply = false);
// Natural-order fused walk with the input generated on the fly (Appendix 1):
// k2_out[r] = k1(perm(start + r)); qubits_struct points to a host
// qsim::Qubits (passed by value as a kernel parameter).
// Layout (host-chosen, kron_layout in qsim_api.cu): pos[k] = address bit at
// table position k; J[0..4] = output bits walked inside a thread (ascending);
// tiles fill aligned blocks of 2^L outputs; nv > 0 enables the per-thread
// hoisted product (source bits at positions >= nv constant in a thread).
int jit_kron(const uint32_t* words, int n, int M, const void* qubits_struct, size_t qbytes,
             int elem, int gbits, int ngroups, const uint8_t* pos, const uint8_t* J, int L, int nv,
             uint64_t start, uint64_t count, void* k2_out, int sms, cudaStream_t st,
             std::string& err);
int jit_check_compile_kron(const uint32_t* words, int n, int M, int elem, int gbits, int ngroups,
                           const uint8_t* pos, const uint8_t* J, int L, int nv, std::string& err);
int jit_check_compile_fused(const uint32_t* words, int n, int M, const uint8_t* sigma, int elem,
                            std::string& err);
// Planned apply from a materialised map (NVRTC; sigma order, the fused
// kernel's batching).  Returns 0 or -1 with err.
int jit_apply(int M, const uint8_t* sigma, uint32_t chunk_log2, int elem, const uint32_t* perm,
              const void* k1, void* k2, void* ticket, int blocks, int warps, cudaStream_t st,
              std::string& err);
int jit_check_compile_apply(int M, const uint8_t* sigma, int elem, std::string& err);
// Circuits whose targets all lie below bit T: tiles of 2^T outputs read their
// own tile of k1, staged in shared memory by TMA bulk copies (double-buffered).
int jit_local(const uint32_t* words, int n, int M, int elem, int T, const void* k1, void* k2,
              uint32_t* perm_out, int sms, cudaStream_t st, std::string& err);
int jit_check_compile_local(const uint32_t* words, int n, int M, int elem, int T, std::string& err);
}  // namespace qsim
