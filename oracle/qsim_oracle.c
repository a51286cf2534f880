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
 * (byte 0 = kind: 0 NOT, 1 CNOT, 2 CCNOT, 3 Z, 4 CZ, 5 CCZ, 6 SWAP; byte 1
 * = target bit b, meaning address bit a(b+1), a(1) the LSB [P:L43 2(b)];
 * bytes 2,3 = control bits, used by CNOT/CZ (byte 2) and CCNOT/CCZ (bytes 2
 * and 3); SWAP exchanges bits byte 1 and byte 2).  Gate 0 is "Step 1" and
 * is applied first (reading R1).
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
 * is symmetric because the toggle is its own inverse.
 *
 * Phase and SWAP steps (reading R17): "Assuming that phase
 * gates are not used, each matrix element produced by a wiring diagram will be
 * non-negative" -- dropping the assumption admits the P:L37 matrix
 * with its -1.  Kind 3 Z, 4 CZ, 5 CCZ: a diagonal step whose row x holds -1
 * when the target bit and every control bit of x are 1, else +1.  Kind 6
 * SWAP: row x has its unity in the column with bits `target` and `c0`
 * exchanged.  Both are symmetric with one non-zero per row.               */
static int oracle_bit(uint64_t x, unsigned b) { return (int)((x >> b) & 1u); }

static int oracle_is_phase(unsigned kind) { return kind >= 3 && kind <= 5; }

int oracle_controls_set(const uint8_t *g, uint64_t x)
{
    unsigned kind = g[0];
    if (kind == 0) return 1;                       /* NOT: no control      */
    if (kind == 1) return oracle_bit(x, g[2]) == 1; /* CNOT: one control   */
    if (kind == 2)                                  /* CCNOT               */
        return oracle_bit(x, g[2]) == 1 && oracle_bit(x, g[3]) == 1;
    if (kind == 3) return 1;                       /* Z: no control        */
    if (kind == 4) return oracle_bit(x, g[2]) == 1;
    if (kind == 5) return oracle_bit(x, g[2]) == 1 && oracle_bit(x, g[3]) == 1;
    return 1;                                      /* SWAP: unconditional  */
}

uint64_t oracle_step(const uint8_t *g, uint64_t x)
{
    unsigned kind = g[0];
    if (oracle_is_phase(kind)) return x;           /* diagonal step        */
    if (kind == 6) {                               /* SWAP bits t, c0      */
        int bt = oracle_bit(x, g[1]), bc = oracle_bit(x, g[2]);
        if (bt != bc) {
            x = bt ? x - ((uint64_t)1 << g[1]) : x + ((uint64_t)1 << g[1]);
            x = bc ? x - ((uint64_t)1 << g[2]) : x + ((uint64_t)1 << g[2]);
        }
        return x;
    }
    if (oracle_controls_set(g, x)) {
        uint64_t target = (uint64_t)1 << g[1];
        if (oracle_bit(x, g[1])) x = x - target; /* target bit 1 -> 0 */
        else                     x = x + target; /* target bit 0 -> 1 */
    }
    return x;
}

/* Diagonal entry of row x of a step: -1 or +1.                           */
int oracle_step_sign(const uint8_t *g, uint64_t x)
{
    if (!oracle_is_phase(g[0])) return 1;
    return (oracle_bit(x, g[1]) == 1 && oracle_controls_set(g, x)) ? -1 : 1;
}

/* ---- composite map, reading R1 (U = U_n ... U_1) and R2 (gather) ---------
 * k2 = U k1.  With U = U_n ... U_1 and each U_k having its non-zero
 * of row x in column f_k(x) with value s_k(x), row i of U has its non-zero
 * in column perm[i] = f_1(f_2( ... f_n(i) ... )) with value
 * sign[i] = s_n(i) s_{n-1}(f_n(i)) ... (each step's entry taken at the
 * address reached so far), i.e. the output address is threaded backwards
 * through the steps, last step first ("calculate a state vector from top to
 * bottom").                                                        */
uint64_t oracle_walk_signed(const uint8_t *gates, int32_t n_gates, uint64_t i, int *sign)
{
    uint64_t x = i;
    int s = 1;
    for (int32_t k = n_gates - 1; k >= 0; --k) {
        const uint8_t *g = gates + 4 * (size_t)k;
        s *= oracle_step_sign(g, x);
        x = oracle_step(g, x);
    }
    *sign = s;
    return x;
}

uint64_t oracle_walk(const uint8_t *gates, int32_t n_gates, uint64_t i)
{
    int s;
    return oracle_walk_signed(gates, n_gates, i, &s);
}

/* Materialised composite ("save information about the unitary matrix",
 * P:L59): perm[i] for every i in [start, start+count).                    */
void oracle_build(const uint8_t *gates, int32_t n_gates,
                  uint64_t start, uint64_t count, uint32_t *perm)
{
    for (uint64_t r = 0; r < count; ++r)
        perm[r] = (uint32_t)oracle_walk(gates, n_gates, start + r);
}

/* ... with the row values of a phased permutation: bit r % 32 of
 * signs[r / 32] is 1 when sign[start + r] = -1 (words fully rewritten).   */
void oracle_build_signed(const uint8_t *gates, int32_t n_gates, uint64_t start,
                         uint64_t count, uint32_t *perm, uint32_t *signs)
{
    for (uint64_t w = 0; w < (count + 31) / 32; ++w) signs[w] = 0;
    for (uint64_t r = 0; r < count; ++r) {
        int s;
        perm[r] = (uint32_t)oracle_walk_signed(gates, n_gates, start + r, &s);
        if (s < 0) signs[r / 32] |= (uint32_t)1 << (r % 32);
    }
}

/* IEEE negation of one complex entry (both parts), as raw bytes.          */
static void oracle_negate(unsigned char *e, int32_t elem_bytes)
{
    if (elem_bytes == 8) {
        float v[2];
        memcpy(v, e, 8);
        v[0] = -v[0];
        v[1] = -v[1];
        memcpy(e, v, 8);
    } else {
        double v[2];
        memcpy(v, e, 16);
        v[0] = -v[0];
        v[1] = -v[1];
        memcpy(e, v, 16);
    }
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

/* Phased form: k2[i] = sign[i] * k1[perm[i]] (signs bitmap as above).     */
void oracle_apply_signed(const uint32_t *perm, const uint32_t *signs, uint64_t count,
                         int32_t elem_bytes, const void *k1, void *k2)
{
    unsigned char *dst = (unsigned char *)k2;
    oracle_apply(perm, count, elem_bytes, k1, k2);
    for (uint64_t i = 0; i < count; ++i)
        if ((signs[i / 32] >> (i % 32)) & 1u) oracle_negate(dst + i * (size_t)elem_bytes, elem_bytes);
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
        int s;
        uint64_t j = oracle_walk_signed(gates, n_gates, start + r, &s);
        memcpy(dst + r * (size_t)elem_bytes, src + j * (size_t)elem_bytes,
               (size_t)elem_bytes);
        if (s < 0) oracle_negate(dst + r * (size_t)elem_bytes, elem_bytes);
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
 * bit-flip step exchanges the two amplitudes of every address pair {x, x
 * with the target toggled} whose control bits are all 1 -- exactly the
 * symmetric unity pattern of the step matrix; a SWAP step exchanges
 * the pairs {x, x with bits t and c0 exchanged}; a phase step negates the
 * amplitudes of the rows whose diagonal entry is -1.  This is the second,
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
            if (oracle_is_phase(g[0])) {
                if (oracle_step_sign(g, x) < 0) oracle_negate(a + x * (size_t)elem_bytes, elem_bytes);
                continue;
            }
            if (g[0] == 6) {
                if (!(oracle_bit(x, g[1]) == 1 && oracle_bit(x, g[2]) == 0)) continue;
            } else {
                if (oracle_bit(x, g[1]) != 0) continue;   /* visit each pair once */
                if (!oracle_controls_set(g, x)) continue; /* row is on diagonal  */
            }
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
        int s;
        const uint64_t j = oracle_walk_signed(gates, n_gates, start + r, &s);
        oracle_kron_element(qubits, M, j, out + 2 * r, out + 2 * r + 1);
        if (s < 0) {
            out[2 * r] = -out[2 * r];
            out[2 * r + 1] = -out[2 * r + 1];
        }
    }
}

int oracle_abi_version(void) { return 1; }
