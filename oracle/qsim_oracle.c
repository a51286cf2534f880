/*
 * qsim_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of what the hot path of
 * Burger, "New approaches to quantum computer simulation in a classical
 * supercomputer" (arXiv quant-ph/0308158) computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or helper with
 * the CUDA product path (paper_quant_ph_0308158_b200/); it has its own gate
 * reader and its own arithmetic.
 *
 * Citations: "P:Lnn" = /root/reference/PAPER.md line nn (section in
 * brackets); readings of silent/garbled passages are the DESIGN.md readings
 * R1..R16 (same numbering as SURVEY.md section 8(c), c1..c16).
 *
 * Gate record (own reader): 4 bytes per gate, in wiring-diagram order
 * (byte 0 = kind: 0 NOT, 1 CNOT, 2 CCNOT; byte 1 = target bit b, meaning
 * address bit a(b+1), a(1) the LSB [P:L43 2(b)]; bytes 2,3 = control bits,
 * used by CNOT (byte 2) and CCNOT (bytes 2 and 3)).  Gate 0 is "Step 1"
 * and is applied first (reading R1).
 *
 * Parity pins for every function: tests/test_oracle_pins.py (worked example
 * P:L43, involution/symmetry P:L39, dense Kronecker products for M<=4,
 * bijection/norm P:L35, the accumulation method P:L59, closed forms, group
 * identities).
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

/* ---- one wiring-diagram step, P:L39 / P:L43 ------------------------------
 * "In Step 1, a(1) is the target bit and a(2) is the controlling bit ...
 * Assuming eight addresses, each is modified, for example, 011 to 010."
 * (P:L43 2(b)).  Generalised to any target and 0, 1 or 2 controls
 * (readings R4, R5): the address x is modified by toggling its target bit
 * when every control bit of x is 1; otherwise x is unchanged.  The step
 * matrix has row x with its single unity in column oracle_step(g, x), which
 * is symmetric because the toggle is its own inverse.              */
static int oracle_bit(uint64_t x, unsigned b) { return (int)((x >> b) & 1u); }

int oracle_controls_set(const uint8_t *g, uint64_t x)
{
    unsigned kind = g[0];
    if (kind == 0) return 1;                       /* NOT: no control      */
    if (kind == 1) return oracle_bit(x, g[2]) == 1; /* CNOT: one control   */
    return oracle_bit(x, g[2]) == 1 && oracle_bit(x, g[3]) == 1; /* CCNOT */
}

uint64_t oracle_step(const uint8_t *g, uint64_t x)
{
    if (oracle_controls_set(g, x)) {
        uint64_t target = (uint64_t)1 << g[1];
        if (oracle_bit(x, g[1])) x = x - target; /* target bit 1 -> 0 */
        else                     x = x + target; /* target bit 0 -> 1 */
    }
    return x;
}

/* ---- composite map, reading R1 (U = U_n ... U_1) and R2 (gather) ---------
 * k2 = U k1.  With U = U_n ... U_1 and each U_k having its unity of
 * row x in column f_k(x), row i of U has its unity in column
 *     perm[i] = f_1(f_2( ... f_n(i) ... )),
 * i.e. the output address is threaded backwards through the steps, last
 * step first ("calculate a state vector from top to bottom").      */
uint64_t oracle_walk(const uint8_t *gates, int32_t n_gates, uint64_t i)
{
    uint64_t x = i;
    for (int32_t k = n_gates - 1; k >= 0; --k)
        x = oracle_step(gates + 4 * (size_t)k, x);
    return x;
}

/* Materialised composite ("save information about the unitary matrix",
 * P:L59): perm[i] for every i in [start, start+count).                    */
void oracle_build(const uint8_t *gates, int32_t n_gates,
                  uint64_t start, uint64_t count, uint32_t *perm)
{
    for (uint64_t r = 0; r < count; ++r)
        perm[r] = (uint32_t)oracle_walk(gates, n_gates, start + r);
}

/* Apply: k2[i] = sum_j U[i][j] k1[j] = k1[perm[i]] because row i of U has a
 * single unity in column perm[i].  Entries are copied as bytes
 * (elem_bytes = 8 for complex64, 16 for complex128), reading R15.         */
void oracle_apply(const uint32_t *perm, uint64_t count, int32_t elem_bytes,
                  const void *k1, void *k2)
{
    const unsigned char *src = (const unsigned char *)k1;
    unsigned char *dst = (unsigned char *)k2;
    for (uint64_t i = 0; i < count; ++i)
        memcpy(dst + i * (size_t)elem_bytes,
               src + (size_t)perm[i] * (size_t)elem_bytes, (size_t)elem_bytes);
}

/* Fused: the same result without storing perm -- the map is recomputed per
 * output ("trading memory for processing").  Output entries
 * [start, start+count) of k2 ("continuous portions").              */
void oracle_fused(const uint8_t *gates, int32_t n_gates,
                  uint64_t start, uint64_t count, int32_t elem_bytes,
                  const void *k1, void *k2_chunk)
{
    const unsigned char *src = (const unsigned char *)k1;
    unsigned char *dst = (unsigned char *)k2_chunk;
    for (uint64_t r = 0; r < count; ++r) {
        uint64_t j = oracle_walk(gates, n_gates, start + r);
        memcpy(dst + r * (size_t)elem_bytes, src + j * (size_t)elem_bytes,
               (size_t)elem_bytes);
    }
}

/* Sampled outputs for full-size parity: src[r] = perm[idx[r]].             */
void oracle_walk_many(const uint8_t *gates, int32_t n_gates,
                      const uint64_t *idx, uint64_t count, uint64_t *src)
{
    for (uint64_t r = 0; r < count; ++r)
        src[r] = oracle_walk(gates, n_gates, idx[r]);
}

/* ---- the "basic accumulation method that avoids the unitary matrix"
 * (P:L59): the state is updated in place gate by gate, Step 1 first.  A
 * step exchanges the two amplitudes of every address pair {x, x with the
 * target toggled} whose control bits are all 1 -- exactly the symmetric
 * unity pattern of the step matrix.  This is the second,
 * algorithmically distinct oracle: no per-address walk, no perm.          */
void oracle_accumulate(const uint8_t *gates, int32_t n_gates, int32_t M,
                       int32_t elem_bytes, void *k)
{
    unsigned char *a = (unsigned char *)k;
    unsigned char tmp[16];
    uint64_t N = (uint64_t)1 << M;
    for (int32_t s = 0; s < n_gates; ++s) {
        const uint8_t *g = gates + 4 * (size_t)s;
        for (uint64_t x = 0; x < N; ++x) {
            if (oracle_bit(x, g[1]) != 0) continue;   /* visit each pair once */
            if (!oracle_controls_set(g, x)) continue; /* row is on diagonal  */
            uint64_t y = oracle_step(g, x);
            memcpy(tmp, a + x * (size_t)elem_bytes, (size_t)elem_bytes);
            memcpy(a + x * (size_t)elem_bytes, a + y * (size_t)elem_bytes,
                   (size_t)elem_bytes);
            memcpy(a + y * (size_t)elem_bytes, tmp, (size_t)elem_bytes);
        }
    }
}

/* ---- Appendix 1: "CALCULATING THE INPUT STATE ON THE FLY" ----
 * "The input can be stored in the form of M qubits labeled q_i, 1 <= i <= M,
 * each represented as a pair of complex numbers [q_i(0) q_i(1)]";
 * k_1 = q_M (x) q_{M-1} (x) ... (x) q_1; "if a particular element
 * ... is wanted, simply use the binary form of i to identify the appropriate
 * components of each qubit to be multiplied. For example, if k_1(5) is
 * wanted, use i = 101 to obtain q_3(1)q_2(0)q_1(1)" ("k_i" read as
 * k_1, reading R12).
 * qubits: 4*M doubles, qubit j (1-based) at [4(j-1)]: re q_j(0), im q_j(0),
 * re q_j(1), im q_j(1).  The product is formed left to right in the order
 * the Kronecker product is written, q_M first, in double precision.        */
void oracle_kron_element(const double *qubits, int32_t M, uint64_t i, double *out_re,
                         double *out_im)
{
    double re = 1.0, im = 0.0;
    for (int32_t j = M; j >= 1; --j) {
        const double *q = qubits + 4 * (size_t)(j - 1) + 2 * (size_t)oracle_bit(i, (unsigned)(j - 1));
        const double r = re * q[0] - im * q[1];
        const double m = re * q[1] + im * q[0];
        re = r;
        im = m;
    }
    *out_re = re;
    *out_im = im;
}

/* Fused with the map: k2[i] = k_1(perm[i]) for the
 * portion [start, start+count); out holds 2*count doubles (re, im).       */
void oracle_fused_kron(const uint8_t *gates, int32_t n_gates, int32_t M, const double *qubits,
                       uint64_t start, uint64_t count, double *out)
{
    for (uint64_t r = 0; r < count; ++r) {
        const uint64_t j = oracle_walk(gates, n_gates, start + r);
        oracle_kron_element(qubits, M, j, out + 2 * r, out + 2 * r + 1);
    }
}

int oracle_abi_version(void) { return 1; }
