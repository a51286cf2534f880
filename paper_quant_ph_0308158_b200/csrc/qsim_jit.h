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
int jit_check_compile(const uint32_t* words, int n, int M, std::string& err);
// Build perm for outputs [start, start+count) with a kernel compiled for this
// exact gate list (per-lane word format).  Returns 0, or -1 with err set (the
// caller then uses the interpreter kernel).
int jit_build(const uint32_t* words, int n, int M, uint64_t start, uint64_t count,
              uint32_t* perm_out, int sms, cudaStream_t st, std::string& err);
}  // namespace qsim
