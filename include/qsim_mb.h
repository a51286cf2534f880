/*
 * qsim_mb.h -- microbenchmarks (libqsim_mb.so), NOT the product path.
 *
 * qsim_mb_gather_c64: k2[r] = k1[idx[r]] for r < count (count % 4 == 0),
 * complex64 entries moved as 8-byte integers, with the k1 gather load issued
 * under cache policy `variant`:
 *   0 ld.global.nc (__ldg)            1 ld.global.cg (L2 only)
 *   2 ld.global.nc.L1::no_allocate    3 ld.global.cs (streaming)
 *   4 ld.global (default .ca)         5 ld.global.L1::no_allocate
 *   6 ld.global.relaxed.gpu           7 ld.global.nc.L1::no_allocate.L2::64B
 * unroll in {1, 2, 4} groups of 4 gathers in flight per thread; blocks <= 0
 * means 148 * 8.  Device pointers, 16-byte aligned.  Returns 0, -1 (bad
 * variant/unroll) or -6 (launch error).  Asynchronous on `stream`.
 */
#ifndef QSIM_MB_H
#define QSIM_MB_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int qsim_mb_gather_c64(const uint32_t *idx, uint64_t count, const void *k1, void *k2,
                       int32_t variant, int32_t unroll, int32_t blocks, void *stream);
/* qsim_mb_tma_gather_c64: the same gather with the TMA engine
 * (cp.async.bulk.tensor tile::gather4, 16-byte rows) into shared memory;
 * stages = producers * 100 + pipeline depth.
 * qsim_mb_scatter_c64: k2[idx[r]] = k1[r] (divergent stores).            */
int qsim_mb_tma_gather_c64(const uint32_t *idx, uint64_t count, const void *k1,
                           uint64_t k1_entries, void *k2, int32_t stages, int32_t blocks,
                           void *stream);
int qsim_mb_scatter_c64(const uint32_t *idx, uint64_t count, const void *k1, void *k2,
                        int32_t unroll, int32_t blocks, void *stream);
#ifdef __cplusplus
}
#endif
#endif
