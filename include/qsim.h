/*
 * qsim.h -- C ABI of libqsim.so, the B200 (sm_100a) hot path of Burger,
 * "New approaches to quantum computer simulation in a classical
 * supercomputer" (arXiv quant-ph/0308158).
 *
 * Citations: "P:Lnn" = PAPER.md line nn (section); R-numbers are the
 * readings of silent / garbled passages listed in DESIGN.md.
 *
 * The method:
 *   - address bits a(M) ... a(1) index the 2^M entries of the state vector,
 *     a(1) the LSB (P:L43 2(b)); here bit b (0-based) is a(b+1) (R3);
 *   - each wiring-diagram step is a 0/1 matrix, symmetric, with one unity
 *     per row: step k maps address x to f_k(x) = x with its target
 *     bit toggled when all its control bits are 1 ("011 to 010"),
 *     for NOT (0 controls), CNOT (1) and CCNOT / Toffoli (2) (R4, R5);
 *   - the composite is U = U_n ... U_1, Step 1 (gates[0]) first (R1); row i
 *     of U has its unity in column perm[i] = f_1(f_2(...f_n(i)...)) (R2);
 *   - the state transform k2 = U k1 is k2[i] = k1[perm[i]],
 *     computed "from top to bottom ... without special sorting".
 *
 * Conventions common to every call
 *   - Status: every call returns QSIM_OK (0) or a negative qsim_status.
 *     Arguments are validated completely BEFORE anything is enqueued, so an
 *     error return means nothing ran.  QSIM_ECUDA means a CUDA API call
 *     failed; qsim_last_error() gives the message (thread-local).
 *   - Asynchrony: device work is enqueued on `stream` (a cudaStream_t; NULL
 *     = legacy default stream) and the call returns without synchronising,
 *     except qsim_run_host (see there).  Faults inside kernels surface at
 *     the caller's next synchronisation.
 *   - Ownership: all buffers are caller-owned.  The library allocates no
 *     device memory for data; the one exception is qsim_run_fused's 256-byte
 *     chunk ticket per (device, stream), allocated on first use and kept for
 *     the life of the process.  `gates` is a host array read during the call
 *     (copied into the launch's kernel-parameter bank); it may be freed on
 *     return.
 *   - Device pointers (perm, k1, k2) must be 16-byte aligned
 *     (QSIM_EINVAL otherwise) and must not overlap each other
 *     (QSIM_EALIAS); all calls are out-of-place.
 *   - Thread safety: reentrant; concurrent calls on different streams are
 *     safe (no mutable module-scope device state).
 *
 * Environment (diagnostics and test switches; none is needed for normal use,
 * none changes a result)
 *   QSIM_NO_JIT=1            never use NVRTC (ahead-of-time kernels only)
 *   QSIM_NVRTC=<path>        libnvrtc to load (default: the toolkit's)
 *   QSIM_JIT_DUMP=<dir>      write each generated kernel source and cubin there
 *   QSIM_THREAD_BITS=0       NVRTC build / on-the-fly input threads walk output
 *                            bits 5..9 (no fast path; same bytes)
 *   QSIM_THREAD_BITS_SAMPLES=k  circuit sample size of the in-thread bits (tests)
 *   QSIM_BUILD_THREAD_BITS=0 build kernel without its in-thread affine fast path
 */
#ifndef QSIM_H
#define QSIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One wiring-diagram step.  kind: 0 NOT, 1 CNOT, 2 CCNOT.
 * target: 0-based bit b, i.e. address bit a(b+1).  c0 (CNOT, CCNOT) and
 * c1 (CCNOT) are the control bits; slots a kind does not use are ignored.
 * Valid: target < M, used controls < M, distinct from the target and from
 * each other.
 *
 * Phased permutations (reading R17: "Assuming that phase gates are
 * not used, each matrix element ... will be non-negative"; the P:L37 matrix
 * has a -1): kind 3 Z, 4 CZ (control c0), 5 CCZ (c0, c1) -- a diagonal step
 * whose row x holds -1 when the target bit and every control bit of x are
 * 1; kind 6 SWAP -- row x has its unity in the column with bits `target` and
 * c0 exchanged.  SWAP is a plain permutation and is accepted everywhere.
 * A circuit with phase steps is a permutation with row values +-1: the calls
 * that produce k2 (run_fused*, run_fused_kron, and build_map_signed +
 * apply_map_signed) apply the -1 as an IEEE negation of both parts (sign
 * bits flipped: bit-exact); the calls whose only output is a uint32 map
 * (build_map*, map_gather_planned, run_host mode 0) return QSIM_EINVAL.      */
typedef struct qsim_gate {
    uint8_t kind;
    uint8_t target;
    uint8_t c0;
    uint8_t c1;
} qsim_gate;

typedef enum qsim_status {
    QSIM_OK     = 0,
    QSIM_EINVAL = -1, /* null / misaligned pointer, bad dtype / mode / kind */
    QSIM_ERANGE = -2, /* M not in [1, 32], or range [start, start+count) not inside [0, 2^M) */
    QSIM_EBIT   = -3, /* a bit >= M, target among controls, duplicate control */
    QSIM_ECAP   = -4, /* n_gates < 0 or > QSIM_MAX_GATES */
    QSIM_EALIAS = -5, /* device buffers overlap */
    QSIM_ECUDA  = -6  /* a CUDA call failed; see qsim_last_error() */
} qsim_status;

typedef enum qsim_dtype {
    QSIM_C64  = 0, /* complex64: 8 bytes per entry (2 x float32)  */
    QSIM_C128 = 1  /* complex128: 16 bytes per entry (2 x float64) */
} qsim_dtype;

/* Largest gate list one launch accepts (the kernel-parameter bank holds
 * 4 bytes per gate, <= 32 KB).                                             */
#define QSIM_MAX_GATES 4096

/* qsim_build_map -- materialise the composite ("save information
 * about the unitary matrix"): perm[i] = f_1(...f_n(i)) for all i < 2^M.
 *   gates   host, n_gates records (may be NULL when n_gates == 0: identity)
 *   M       number of address bits, 1..32
 *   perm    device, 2^M uint32 entries (written)                          */
int qsim_build_map(const qsim_gate *gates, int32_t n_gates, int32_t M,
                   uint32_t *perm, void *stream);

/* Same, for the "continuous portion" [start, start+count):
 * perm_out[r] = perm[start + r].  count may be 0.                          */
int qsim_build_map_range(const qsim_gate *gates, int32_t n_gates, int32_t M,
                         uint64_t start, uint64_t count, uint32_t *perm_out,
                         void *stream);

/* qsim_build_map_signed -- a phased permutation materialised: perm_out[r]
 * as above and its row values, bit r % 32 of signs[r / 32] = 1 when row
 * start + r holds -1 (words of the range fully written; bits past count 0).
 *   start   multiple of 32 (QSIM_EINVAL otherwise); count may be 0
 *   signs   device, (count + 31) / 32 uint32 words, 4-byte aligned       */
int qsim_build_map_signed(const qsim_gate *gates, int32_t n_gates, int32_t M,
                          uint64_t start, uint64_t count, uint32_t *perm_out,
                          uint32_t *signs, void *stream);

/* qsim_apply_map_signed -- k2_out[r] = sign[r] k1[perm_in[r]], r < count,
 * with the bitmap of qsim_build_map_signed (bit r % 32 of signs[r / 32]).  */
int qsim_apply_map_signed(const uint32_t *perm_in, const uint32_t *signs, uint64_t count,
                          int32_t M, int32_t dtype, const void *k1, void *k2_out,
                          void *stream);

/* qsim_apply_map -- the state transform k2 = U k1 given the
 * materialised map: k2[i] = k1[perm[i]] for all i < 2^M.  Entries are
 * moved as raw bytes (bit-exact; -0.0 and NaN payloads preserved).
 *   perm   device, 2^M uint32 (each < 2^M; a permutation if built above)
 *   dtype  QSIM_C64 or QSIM_C128
 *   k1     device, 2^M entries (read)     k2  device, 2^M entries (written)*/
int qsim_apply_map(const uint32_t *perm, int32_t M, int32_t dtype,
                   const void *k1, void *k2, void *stream);

/* Range form: k2_out[r] = k1[perm_in[r]] for r < count; k1 holds all 2^M
 * entries.  perm_in is typically perm + start of a full map.              */
int qsim_apply_map_range(const uint32_t *perm_in, uint64_t count, int32_t M,
                         int32_t dtype, const void *k1, void *k2_out,
                         void *stream);

/* qsim_run_fused -- k2[i] = k1[f_1(...f_n(i))] without storing the map:
 * the memory-for-processing trade-off.  Same arguments as
 * build + apply; no perm buffer.  For M >= 13 with NVRTC the call plans the
 * traversal itself (qsim_plan_create, cached per circuit) and runs the
 * planned kernel with a per-stream chunk ticket -- the same k2 bytes as
 * every other path, at the planned call's speed.                          */
int qsim_run_fused(const qsim_gate *gates, int32_t n_gates, int32_t M,
                   int32_t dtype, const void *k1, void *k2, void *stream);

/* Range form: k2_out[r] = k1[perm[start + r]], r < count.                 */
int qsim_run_fused_range(const qsim_gate *gates, int32_t n_gates, int32_t M,
                         int32_t dtype, uint64_t start, uint64_t count,
                         const void *k1, void *k2_out, void *stream);

/* Walk algorithm selection for build / fused (ablation and tests).
 *   QSIM_WALK_AUTO       library choice: build with >= 2^22 outputs uses the
 *                        circuit-specialised JIT kernel when NVRTC loads
 *                        (compiled once per circuit per process, then
 *                        cached), else the bit-sliced interpreter
 *   QSIM_WALK_PER_LANE   one address per lane, 2 integer ops per gate
 *   QSIM_WALK_BITSLICED  32 addresses per thread, one bit-plane word per
 *                        address bit in shared memory, one logic op per gate */
typedef enum qsim_walk {
    QSIM_WALK_AUTO = 0,
    QSIM_WALK_PER_LANE = 1,
    QSIM_WALK_BITSLICED = 2,
    QSIM_WALK_JIT = 3       /* build only: kernel compiled for this circuit (NVRTC);
                               QSIM_ECUDA if NVRTC is unavailable                */
} qsim_walk;

int qsim_build_map_ex(const qsim_gate *gates, int32_t n_gates, int32_t M,
                      uint64_t start, uint64_t count, uint32_t *perm_out,
                      int32_t walk, void *stream);
int qsim_run_fused_ex(const qsim_gate *gates, int32_t n_gates, int32_t M,
                      int32_t dtype, uint64_t start, uint64_t count,
                      const void *k1, void *k2_out, int32_t walk, void *stream);

/* ---- traversal plans (locality of the gather) ----------------------------
 * The gather reads k1 at perm[i]; in natural output order the readers of one
 * 128-byte line of k1 are scattered over the whole output range, so for a
 * random circuit almost every read misses L2.  A plan orders the traversal:
 * output i = sigma(c) for counter c = 0 .. 2^M-1, sigma a permutation of
 * the address bits that keeps bits 0..2 (complex64) / 0..1 (complex128) in
 * place (stores stay whole 32-byte sectors).  Counter bits 0..tile_log2-1
 * are the "sector cover": the output bits in which the readers of one
 * 32-byte k1 sector most often differ, so they are handled by one CTA close
 * in time and its L1 serves the sector after the first miss; the remaining
 * bits follow in order of how often the readers of one 128-byte k1 line
 * differ in them.  CTAs take chunks of 2^chunk_log2 counters strictly in
 * counter order from a device ticket, so the lines a chunk front touches
 * stay in L2.  The result is the same k2 bytes; only the order of work
 * changes.
 *
 * qsim_plan_create samples the circuit on the host (forward and inverse
 * walks of pseudo-random outputs and k1 lines, fixed seeds: deterministic)
 * and fills `plan`, a plain value owned by the caller.  chunk_log2 and
 * blocks_per_sm may be edited before use (tuning).                          */
#define QSIM_WORKSPACE_BYTES 256
#define QSIM_PLAN_SPLIT 4u  /* qsim_plan.flags bit 2 (below) */

typedef struct qsim_plan {
    int32_t M;
    int32_t dtype;          /* QSIM_C64 / QSIM_C128: a 128-B line holds 16 / 8 entries */
    uint32_t chunk_log2;    /* counters per CTA chunk (default 16), within [10, M] */
    int32_t blocks_per_sm;  /* resident CTAs per SM (default 1), 1..8          */
    uint32_t flags;         /* bit 0: natural order (no sigma): set when the state is
                               L2-resident (<= 64 MB) or when the sector cover holds
                               under 1/4 of the sampled pairs (no order helps).
                               bit 1: the circuit keeps locality -- every target (and
                               SWAP partner) bit is below T = 13 (complex64) / 12
                               (complex128), so each aligned tile of 2^T outputs reads
                               its own tile of k1: map+gather and fused use the
                               shared-memory staged kernel (TMA bulk copies of k1
                               tiles, double-buffered), re-checked on the gates given.
                               bit 2 (QSIM_PLAN_SPLIT, sigma plans only): the map +
                               gather step runs as two kernels -- the planned gather
                               with the map recomputed in registers (k2 only), then
                               the natural-order build (perm in coalesced runs) --
                               instead of one kernel storing perm in plan order;
                               same bytes, set by qsim_plan_tune when it measures
                               faster (the scattered perm runs cost a DRAM row
                               activation each)                                   */
    uint16_t ilp;           /* gathers in flight per thread: 8, 16 or 32 (0 = 16) */
    uint16_t cta_threads;   /* CTA size: 256, 512 or 1024 (0 = 256); the NVRTC
                               gather kernels run 16 warps for 512, else 8     */
    uint16_t fused_chunk_log2; /* counters per CTA chunk of the fused kernel (default 16) */
    uint16_t reserved_spread;  /* diagnostics: log2 of the 0.9-quantile spread of a line's
                                  readers, natural order (low byte) and sigma order (high) */
    uint8_t sigma[32];      /* counter bit k -> output bit sigma[k]            */
    float change_freq[32];  /* per output bit: fraction of sampled k1 lines whose
                               readers differ in that bit                     */
    uint8_t tile_log2;      /* diagnostics (ABI 2): counter bits 0..tile_log2-1 are the
                               "sector cover" -- the output bits in which the readers
                               of one 32-byte k1 sector most often differ (sampled)   */
    uint8_t tile_reserved[3];
    float tile_contained;   /* sampled fraction of (reader, sector-mate reader) pairs
                               that differ only in those bits                        */
} qsim_plan;

int qsim_plan_create(const qsim_gate *gates, int32_t n_gates, int32_t M, int32_t dtype,
                     qsim_plan *plan);

/* qsim_plan_tune -- measure plan variants for this circuit on the caller's
 * buffers (like an FFTW_MEASURE plan) and keep the fastest map + gather:
 * the default cover rule and the full 13-bit cover, each with and without
 * lanes on output bits 0..4, and full covers of 11 and 12 bits (distinct
 * orders only), then chunks of 2^(c-1) / 2^(c+1) counters for the kept order,
 * then the order of the counter bits above the sector cover (every tail bit
 * at each of the 10 positions next to the cover, best move kept on a >= 0.5 %
 * win, up to 3 rounds; sigma[10..] is a kernel parameter, so no recompiles),
 * then exchanges of any two counter positions >= 10 (every pair screened,
 * the four best re-timed, the best kept on a >= 0.5 % win, up to 2 rounds),
 * then exchanges of a compiled position (3..9: lanes and in-thread entries,
 * a new kernel each, a round's kernels compiled in parallel on the host)
 * with any later position, the same way, up to 3 rounds (each kept move
 * followed by one more round of runtime exchanges), then the chunk size
 * (2^(c±1)), 2 CTAs per SM and 512-thread CTAs once more for the kept order.  In every stage the four
 * best screened candidates are re-timed interleaved with the current order
 * (clock drift under sw_power_cap cancels) and the best ratio is kept on a
 * >= 0.5 % win.
 * Each trial runs qsim_map_gather_planned (the first of a variant compiles
 * its kernel), so perm and k2 hold a valid result afterwards; the call
 * synchronises `stream` (cfg5: about 60 s).  plan: in (chunk sizes, residency kept) /
 * out; chosen (may be NULL): index of the variant kept (0 default rule, 1
 * rule + lanes 0..4, 2 full cover, 3 full + lanes, 4/5 full 11/12-bit;
 * + 8: the same order as the two-kernel step, flag QSIM_PLAN_SPLIT -- every
 * sigma variant is also timed that way in the first stage).
 * QSIM_EINVAL for phase circuits (the map + gather step refuses them).     */
int qsim_plan_tune(qsim_plan *plan, const qsim_gate *gates, int32_t n_gates, uint32_t *perm,
                   const void *k1, void *k2, void *workspace, void *stream, int32_t *chosen);

/* qsim_plan_tune_ex -- qsim_plan_tune with a search effort (like FFTW's
 * planner flags):
 *   QSIM_TUNE_MEASURE  stages 1-3 (cover variants, chunk size, moves of the
 *                      runtime counter bits): cfg5 about 10 s, 19.1-19.3 ms
 *   QSIM_TUNE_PATIENT  all six stages (= qsim_plan_tune): cfg5 about 60 s,
 *                      17.6-18.0 ms (profiles/r02_tune_trace_cfg5.txt)
 * Any other effort: QSIM_EINVAL (nothing runs).  The kernels compiled for
 * the candidates stay in the process's JIT cache (PATIENT at M = 32: about
 * 500 modules of tens of KB of device code each).                          */
enum { QSIM_TUNE_MEASURE = 1, QSIM_TUNE_PATIENT = 2,
       QSIM_TUNE_APPLY = 0x100 /* OR-ed into effort: tune qsim_apply_map_planned
                                  instead -- perm is built first (the map of gates),
                                  the trials time the planned apply on it (k2
                                  written); the two-kernel form is not tried   */ };
int qsim_plan_tune_ex(qsim_plan *plan, const qsim_gate *gates, int32_t n_gates, uint32_t *perm,
                      const void *k1, void *k2, void *workspace, void *stream, int32_t effort,
                      int32_t *chosen);

/* qsim_apply_map_planned -- qsim_apply_map (the same k2, bit for bit) in the
 * traversal order of `plan` (M and dtype are plan->M, plan->dtype).
 *   workspace  device scratch of QSIM_WORKSPACE_BYTES (16-B aligned), reset
 *              on `stream` by the call; must not be used by a concurrent
 *              call.  NULL: grid-stride chunk order (slower, still correct).
 * QSIM_EINVAL if the plan is malformed (sigma not a permutation of 0..M-1
 * fixing bits 0..2 / 0..1, chunk_log2 or blocks_per_sm out of range).      */
int qsim_apply_map_planned(const qsim_plan *plan, const uint32_t *perm, const void *k1,
                           void *k2, void *workspace, void *stream);

/* qsim_run_fused_planned -- qsim_run_fused (the same k2) with the walk done
 * for the outputs in the plan's order; `gates` must be the circuit the plan
 * was created from (same n_gates; the plan is not re-derived).  With a
 * workspace and NVRTC the kernel is compiled for (circuit, sigma, dtype) on
 * first use and cached for the process.                                      */
int qsim_run_fused_planned(const qsim_plan *plan, const qsim_gate *gates, int32_t n_gates,
                           const void *k1, void *k2, void *workspace, void *stream);

/* qsim_run_fused_kron -- the state transform with the INPUT GENERATED ON THE
 * FLY (Appendix 1): k1 is never stored; it is the Kronecker
 * product k1 = q_M (x) ... (x) q_1 of M qubits [q_j(0) q_j(1)] (P:L81,
 * P:L83), so k1(s) = q_M(b_M) ... q_1(b_1) for s = b_M...b_1 ("use i = 101
 * to obtain q_3(1)q_2(0)q_1(1)"), and
 *     k2_out[r] = k1(perm[start + r]),   r < count.
 *   qubits  host, 4*M doubles: qubit j (1-based) at [4(j-1)]: re q_j(0),
 *           im q_j(0), re q_j(1), im q_j(1); rounded to the state precision
 *           (float for QSIM_C64) before use
 *   M       1..63: the only call that accepts M > 32 -- k1 is never stored,
 *           so only the output portion [start, start+count) needs memory
 *           ("output in convenient continuous portions"; "a quantum
 *           computer of 64 qubits ... impossible to store").  For
 *           M > 32 addresses are 64-bit (64 bit planes in the NVRTC kernel)
 *   k2_out  device, count entries of dtype (written)
 *   walk    QSIM_WALK_AUTO / QSIM_WALK_BITSLICED / QSIM_WALK_JIT, or
 *           QSIM_WALK_PER_LANE (one 64-bit address per lane; the fallback
 *           for M > 32 without NVRTC, where BITSLICED means PER_LANE)
 * Arithmetic: the factors are grouped by bits of s into ng tables of
 * products of gb qubits each (descending table position; complex64: gb <= 10, e.g. 4
 * groups of 8 bits at M = 32, 4 of 10 at M = 40; complex128: gb <= 8), combined from the top
 * group down, ((T_{ng-1} T_{ng-2}) ...) T_0 -- the same in every walk.  Which
 * address bits form which group is chosen per call by sampling the circuit
 * (the in-thread layout: table 0 holds the few source bits that vary across
 * an NVRTC thread's 32 outputs, the product of the other groups is formed
 * once per thread); every kernel of a call uses that grouping, so the walks
 * give identical bytes, and the grouping of a call is deterministic.  Every
 * complex product is re = fma(ar, br, -(ai*bi)), im = fma(ar, bi, ai*br)
 * (the inner products rounded, then one fused rounding).  Not bit-exact
 * against a sequential double product: each complex product has normwise
 * relative error <= 2u with an FMA (Jeannerod, Kornerup, Louvet & Muller
 * 2017), so M - 1 products stay within (M-1)*sqrt(5)*u (u = 2^-24 for
 * complex64, 2^-53 for complex128), the tolerance the tests use.          */
int qsim_run_fused_kron(const qsim_gate *gates, int32_t n_gates, int32_t M, int32_t dtype,
                        const double *qubits, uint64_t start, uint64_t count, void *k2_out,
                        int32_t walk, void *stream);

/* qsim_map_gather_planned -- materialised map AND gather in one call:
 * perm[i] = f_1(...f_n(i)) for all i (natural layout, as qsim_build_map) and
 * k2[i] = k1[perm[i]] (as qsim_apply_map).  With a sigma plan, a workspace
 * and NVRTC available this is ONE kernel compiled for the circuit that
 * walks each output once, stores its map entry and gathers (no re-read of
 * perm); otherwise it is qsim_build_map followed by the planned gather.    */
int qsim_map_gather_planned(const qsim_plan *plan, const qsim_gate *gates, int32_t n_gates,
                            uint32_t *perm, const void *k1, void *k2, void *workspace,
                            void *stream);

/* qsim_run_host -- the whole path from HOST buffers (end-to-end use):
 * copies k1_host -> k1_dev, computes k2 (mode 0: qsim_map_gather_planned,
 * the map materialised in perm_dev; mode 1: planned fused, perm_dev unused
 * and may be NULL), copies k2_dev -> k2_host, and SYNCHRONISES `stream`
 * before returning.  The plan is created inside the call (host sampling,
 * ~1-3 ms); the first call for a circuit also JIT-compiles its kernel.
 *   k1_host, k2_host  host, 2^M entries each (pinned memory recommended)
 *   k1_dev, k2_dev    device workspaces, 2^M entries each
 *   perm_dev          device workspace, 2^M uint32 (mode 0)
 *   workspace         device, QSIM_WORKSPACE_BYTES (may be NULL)           */
int qsim_run_host(const qsim_gate *gates, int32_t n_gates, int32_t M,
                  int32_t dtype, int32_t mode, const void *k1_host,
                  void *k2_host, void *k1_dev, void *k2_dev,
                  uint32_t *perm_dev, void *workspace, void *stream);

/* qsim_run_host_batch -- nsteps independent states end to end, with the
 * copies overlapped (serving): step i copies k1_hosts[i] in, computes k2 as
 * qsim_run_host (mode 0 / 1), copies it to k2_hosts[i]; step i+1's copy in
 * and step i-1's copy out run while step i computes (PCIe is full duplex).
 * Double-buffered device state: step i uses k1_dev{i&1}, k2_dev{i&1} (2^M
 * entries each, e.g. 4 x 32 GiB + a 16 GiB map at M = 32).  One plan for
 * all steps; library-created streams; SYNCHRONISES before returning.
 * k1_hosts / k2_hosts: nsteps host pointers each (may repeat; pinned
 * memory recommended).                                                     */
int qsim_run_host_batch(const qsim_gate *gates, int32_t n_gates, int32_t M, int32_t dtype,
                        int32_t mode, int32_t nsteps, const void *const *k1_hosts,
                        void *const *k2_hosts, void *k1_dev0, void *k1_dev1, void *k2_dev0,
                        void *k2_dev1, uint32_t *perm_dev, void *workspace);

/* CUDA graphs for launch-bound loops (small states: a 2^20-entry step runs
 * in a few microseconds, less than its host-side launch path).
 * qsim_graph_create records `reps` consecutive steps of one planned call --
 * call 0: qsim_map_gather_planned, 1: qsim_run_fused_planned, 2:
 * qsim_apply_map_planned -- on the given buffers into a CUDA graph (after one
 * uncaptured step that validates the arguments and compiles the kernels; it
 * synchronises).  qsim_graph_launch replays all reps on `stream`
 * (asynchronous; the buffers must stay alive and unchanged in place);
 * qsim_graph_destroy frees it.  `plan` and `gates` are read during create
 * only.  reps in [1, 1024]; errors as the recorded call.                   */
typedef struct qsim_graph qsim_graph;
int qsim_graph_create(const qsim_plan *plan, const qsim_gate *gates, int32_t n_gates, int32_t call,
                      uint32_t *perm, const void *k1, void *k2, void *workspace, int32_t reps,
                      qsim_graph **out);
int qsim_graph_launch(qsim_graph *graph, void *stream);
int qsim_graph_destroy(qsim_graph *graph);

/* Number of kernel launches the last successful call on this thread
 * enqueued (for launch accounting in bench.py).                            */
int32_t qsim_last_launch_count(void);
/* Name of the last kernel the last planned call, build_map or run_fused_kron
 * call on this thread launched ("qsim_jit_fused", "k_fused_sigma",
 * "qsim_jit_build (J 7.8.13.26.29, L 32, nv 5)" -- the in-thread output bits,
 * block size and varying source bits --, ...; "" if none).                 */
const char *qsim_last_kernel(void);

const char *qsim_strerror(int32_t code);
const char *qsim_last_error(void);
/* JIT diagnostics: "ready", or why the JIT path is unavailable; duration of
 * the most recent NVRTC compile (0 if none).                               */
const char *qsim_jit_status(void);
double qsim_jit_last_compile_ms(void);
/* NVRTC-compiles (does not load or launch) the circuit-specialised build
 * kernel for this gate list; works without a GPU.  QSIM_ECUDA with the
 * NVRTC log in qsim_last_error() on failure.                               */
int qsim_jit_check_compile(const qsim_gate *gates, int32_t n_gates, int32_t M);
/* Same for the sigma-ordered fused / map+gather kernel of a plan, and for the
 * Appendix-1 (input on the fly) kernel.                                     */
int qsim_jit_check_compile_kron(const qsim_gate *gates, int32_t n_gates, int32_t M,
                                int32_t dtype);
int qsim_jit_check_compile_planned(const qsim_plan *plan, const qsim_gate *gates,
                                   int32_t n_gates);
/* ABI version of this header / library: 7 (plans with the sector cover,
 * phase / SWAP gates, M > 32 on-the-fly input, batch e2e, graphs, tuning;
 * 7: the measured-slower linear-traversal and lane-pair plan fields removed). */
int32_t qsim_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QSIM_H */
