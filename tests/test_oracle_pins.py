"""Pin the CPU oracle to things other than itself (CPU only, -m "not gpu").

Each test names what it pins and where that comes from.  "P:Lnn" is a
PAPER.md line; R-numbers are DESIGN.md readings.  A plausible mistake in the
oracle -- a dropped control, a wrong target index, walking the steps in the
wrong order, gather/scatter swapped, a transposed operand -- fails at least
one of these:

* worked example, Toffoli truth table (textbook)  -> step semantics
* dense Kronecker construction, exhaustive over all gates for M <= 4
  -> bit index / control handling (independent construction)
* dense composite products U_n...U_1 for M <= 4 and the P:L37 matrix
  -> composition order and gather direction (R1, R2)
* the accumulation method -> whole-vector result at M up to 14
* closed forms (NOT-only XOR mask; NOT/CNOT affine over GF(2)), group
  identities, bijection and norm, empty / repeated gates.
"""
import os

import numpy as np
import pytest

import oracle
import oracle.dense as dense
import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def _all_gates(M):
    gs = []
    for t in range(M):
        gs.append(wl.gate(wl.NOT, t))
        for c in range(M):
            if c != t:
                gs.append(wl.gate(wl.CNOT, t, c))
        for c0 in range(M):
            for c1 in range(c0 + 1, M):
                if t not in (c0, c1):
                    gs.append(wl.gate(wl.CCNOT, t, c0, c1))
    return gs


# ---------------------------------------------------------------- step level
def test_worked_example_P43():
    (M, t, c, a_in, a_out), = _rows("worked_step_P43.txt")
    g = wl.gate(wl.CNOT, int(t), int(c))
    assert oracle.step(g, int(a_in, 2)) == int(a_out, 2)      # 011 -> 010
    assert oracle.step(g, int(a_out, 2)) == int(a_in, 2)      # symmetric partner
    # the control a(2) not asserted: identity branch
    assert oracle.step(g, 0b001) == 0b001
    assert oracle.step(g, 0b101) == 0b101
    # full 8-address step map: exactly the rows with a(2)=1 swap a(1)
    assert [oracle.step(g, x) for x in range(8)] == [0, 1, 3, 2, 4, 5, 7, 6]
    assert wl.worked_step().tolist() == g.tolist()


def test_toffoli_truth_table():
    g = wl.gate(wl.CCNOT, 0, 2, 1)
    for a_in, a_out in _rows("toffoli_truth_table.txt"):
        assert oracle.step(g, int(a_in, 2)) == int(a_out, 2)


@pytest.mark.parametrize("M", [1, 2, 3, 4])
def test_step_equals_kronecker_matrix_exhaustive(M):
    """Every gate on M <= 4 bits: row x of the textbook Kronecker-product
    matrix has its unity in column step(x); the matrix is symmetric,
    non-negative and has one unity per row."""
    for g in _all_gates(M):
        S = dense.step_matrix(g, M)
        assert np.all(S >= 0)
        assert np.array_equal(S, S.T)
        assert np.all(S.sum(axis=1) == 1) and np.all((S == 0) | (S == 1))
        cols = [oracle.step(g, x) for x in range(1 << M)]
        assert np.array_equal(dense.perm_of(S), np.array(cols, dtype=np.uint32))


def test_step_is_involution():
    rng = np.random.default_rng(7)
    for M in (5, 10, 32):
        for g in wl.random_gates(20, M, int(rng.integers(1 << 30))):
            for x in rng.integers(0, 1 << M, size=64, dtype=np.uint64):
                y = oracle.step(g, int(x))
                assert oracle.step(g, y) == int(x)
                # only the target bit may change
                assert (y ^ int(x)) in (0, 1 << int(g[1]))


# ------------------------------------------------------------ composite level
@pytest.mark.parametrize("M", [1, 2, 3, 4])
def test_composite_equals_dense_product(M):
    """R1/R2: perm == rows of U_n...U_1 built from Kronecker products, and
    k2 == U @ k1 by value."""
    for seed in range(40):
        n = [0, 1, 2, 5, 9, 17][seed % 6]
        if M == 1:
            gates = wl.gates_array([wl.gate(wl.NOT, 0)] * (seed % 3))
        elif M == 2:
            rng = np.random.default_rng(seed)
            gates = wl.gates_array([wl.gate(wl.NOT, int(rng.integers(2))) if rng.integers(2)
                                    else wl.gate(wl.CNOT, *map(int, rng.permutation(2)))
                                    for _ in range(n)])
        else:
            gates = wl.random_gates(n, M, seed)
        U = dense.composite_matrix(gates, M)
        perm = oracle.build_map(gates, M)
        assert np.array_equal(dense.perm_of(U), perm)
        k1 = wl.make_state(wl.StateSpec(M, "c128", wl.GAUSS, seed))
        k2 = oracle.apply_map(perm, k1)
        np.testing.assert_array_equal(U @ k1, k2)       # by value (R15)
        # unitarity of the dense product
        np.testing.assert_array_equal(U.T @ U, np.eye(1 << M))


def test_paper_matrix_P37_direction():
    """The P:L37 matrix is unitary; its entrywise absolute value is the
    composite of [CNOT(t=a(2),c=a(1)), NOT(a(2)), CNOT(t=a(1),c=a(2)),
    NOT(a(2))] under the gather reading (R2) -- the scatter reading would
    give the transpose."""
    rows = _rows("example_matrix_P37.txt")
    P = np.zeros((4, 4))
    for r, c, v in rows:
        P[int(r), int(c)] = float(v)
    np.testing.assert_array_equal(P.T @ P, np.eye(4))
    assert not np.array_equal(np.abs(P), np.abs(P).T)   # not a single step
    gates = wl.gates_array([wl.gate(wl.CNOT, 1, 0), wl.gate(wl.NOT, 1),
                            wl.gate(wl.CNOT, 0, 1), wl.gate(wl.NOT, 1)])
    assert np.array_equal(dense.composite_matrix(gates, 2), np.abs(P))
    assert oracle.build_map(gates, 2).tolist() == [3, 0, 2, 1]


def test_cfg1_golden():
    """Regression fixture written by tests/golden/make_golden.py (oracle only)."""
    rows = _rows("cfg1_perm.txt")
    want = [int(v) for v in rows[0]]
    got = oracle.build_map(wl.CONFIGS["cfg1"].gates(), 3).tolist()
    assert got == want
    U = dense.composite_matrix(wl.CONFIGS["cfg1"].gates(), 3)
    assert dense.perm_of(U).tolist() == want


@pytest.mark.parametrize("M", [3, 8, 12, 14])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_accumulation_method_equals_composite(M, dtype):
    """P:L59's "basic accumulation method" (gate-by-gate pair swaps, no
    per-address walk) gives the same bytes as build + apply."""
    gates = wl.random_gates(48, M, 100 + M)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, M))
    k2 = oracle.apply_map(oracle.build_map(gates, M), k1)
    acc = oracle.accumulate(gates, k1)
    assert acc.tobytes() == k2.tobytes()
    # a ripple cascade too (structured, carries)
    rg = wl.ripple_gates(M, 40) if M >= 3 else gates
    assert oracle.accumulate(rg, k1).tobytes() == oracle.apply_map(
        oracle.build_map(rg, M), k1).tobytes()


@pytest.mark.parametrize("M", [1, 6, 16])
def test_bijection_and_norm(M):
    gates = wl.random_gates(64, M, M) if M >= 3 else wl.gates_array([wl.gate(wl.NOT, 0)])
    perm = oracle.build_map(gates, M)
    assert np.array_equal(np.sort(perm), np.arange(1 << M, dtype=np.uint32))
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 5))
    k2 = oracle.apply_map(perm, k1)
    # same multiset of bit patterns => identical norm, exactly
    assert np.array_equal(np.sort(k1.view(np.uint64)), np.sort(k2.view(np.uint64)))


def test_not_only_closed_form():
    """NOT-only circuit: perm[i] = i XOR (targets with odd multiplicity)."""
    rng = np.random.default_rng(3)
    M = 12
    ts = rng.integers(0, M, size=31)
    gates = wl.gates_array([wl.gate(wl.NOT, int(t)) for t in ts])
    mask = 0
    for t in ts:
        mask ^= 1 << int(t)
    assert np.array_equal(oracle.build_map(gates, M),
                          np.arange(1 << M, dtype=np.uint32) ^ np.uint32(mask))


def test_not_cnot_affine_closed_form():
    """NOT/CNOT circuits are affine over GF(2): perm[i] = A i + b with
    b = perm[0] and column j of A = perm[2^j] XOR perm[0]."""
    M = 11
    rng = np.random.default_rng(11)
    rows = []
    for _ in range(60):
        if rng.integers(2):
            rows.append(wl.gate(wl.NOT, int(rng.integers(M))))
        else:
            t, c = rng.choice(M, 2, replace=False)
            rows.append(wl.gate(wl.CNOT, int(t), int(c)))
    gates = wl.gates_array(rows)
    perm = oracle.build_map(gates, M)
    b = int(perm[0])
    cols = [int(perm[1 << j]) ^ b for j in range(M)]
    for i in range(1 << M):
        v = b
        for j in range(M):
            if (i >> j) & 1:
                v ^= cols[j]
        assert int(perm[i]) == v
    # a Toffoli breaks affinity somewhere (the test can tell)
    perm2 = oracle.build_map(wl.gates_array(rows + [wl.gate(wl.CCNOT, 0, 1, 2)]), M)
    b2 = int(perm2[0])
    cols2 = [int(perm2[1 << j]) ^ b2 for j in range(M)]
    assert int(perm2[0b111]) != b2 ^ cols2[0] ^ cols2[1] ^ cols2[2]


@pytest.mark.parametrize("M", [10, 20])
def test_group_identities(M):
    """G ++ reverse(G) is the identity; perm(reverse G) is perm(G)^-1."""
    gates = wl.random_gates(64, M, 40 + M)
    rev = gates[::-1].copy()
    ident = oracle.build_map(np.concatenate([gates, rev]), M)
    assert np.array_equal(ident, np.arange(1 << M, dtype=np.uint32))
    p, q = oracle.build_map(gates, M), oracle.build_map(rev, M)
    assert np.array_equal(q[p], np.arange(1 << M, dtype=np.uint32))


def test_group_identity_at_32_bits_sampled():
    gates = wl.CONFIGS["cfg5"].gates()
    idx = np.random.default_rng(0).integers(0, 1 << 32, size=4096, dtype=np.uint64)
    src = oracle.walk_many(gates, idx)
    assert src.max() < (1 << 32)
    back = oracle.walk_many(gates[::-1].copy(), src)
    assert np.array_equal(back, idx)


def test_empty_and_repeated_gates():
    M = 9
    ident = np.arange(1 << M, dtype=np.uint32)
    assert np.array_equal(oracle.build_map(np.zeros((0, 4), np.uint8), M), ident)
    for g in wl.random_gates(10, M, 9):
        assert np.array_equal(oracle.build_map(wl.gates_array([g, g]), M), ident)


def test_fused_and_chunks_equal_materialised():
    M = 13
    gates = wl.random_gates(64, M, 77)
    for dtype in ("c64", "c128"):
        k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 3))
        full = oracle.apply_map(oracle.build_map(gates, M), k1)
        assert oracle.run_fused(gates, k1).tobytes() == full.tobytes()
        cuts = [0, 1, 100, 4096, 5000, 1 << M]
        glued = np.concatenate([oracle.run_fused(gates, k1, a, b - a)
                                for a, b in zip(cuts[:-1], cuts[1:])])
        assert glued.tobytes() == full.tobytes()
        part = oracle.build_map(gates, M, 4000, 300)
        assert np.array_equal(part, oracle.build_map(gates, M)[4000:4300])


def test_high_bits_untouched_by_low_circuit():
    """Gates confined to bits < 8 move entries only inside 256-entry blocks."""
    M = 16
    gates = wl.random_gates(50, 8, 5)
    perm = oracle.build_map(gates, M).astype(np.int64)
    assert np.array_equal(perm >> 8, np.arange(1 << M) >> 8)


# ------------------------------------------------ Appendix 1 (input on the fly)
def test_appendix1_worked_example_P89():
    """k_1(5) with i = 101 is q_3(1) q_2(0) q_1(1)."""
    (tag, M, ibits, *factors), = _rows("appendix1_P87_P89.txt")
    M, i = int(M), int(ibits, 2)
    q = wl.random_qubits(M, 11, "c128")
    want = 1.0 + 0j
    for f in factors:
        j, c = map(int, f.split(":"))
        want *= q[j - 1, c]
    assert abs(oracle.kron_element(q, i) - want) <= 1e-15 * abs(want)


@pytest.mark.parametrize("M", [1, 3, 7])
def test_appendix1_all_ones_P87(M):
    """Every qubit |1> = [0 1]: the Kronecker product is the basis vector of
    the all-ones address 2^M - 1 (reading R12)."""
    q = wl.basis_qubits(M, 1, "c128")
    vals = [oracle.kron_element(q, i) for i in range(1 << M)]
    assert vals[(1 << M) - 1] == 1
    assert all(v == 0 for v in vals[:-1])


@pytest.mark.parametrize("M", [1, 2, 5, 10])
def test_appendix1_equals_numpy_kron(M):
    """Element-wise generation equals the full Kronecker product built with
    numpy.kron in the written order q_M (x) ... (x) q_1."""
    q = wl.random_qubits(M, 100 + M, "c128")
    full = np.ones(1, dtype=np.complex128)
    for j in range(M, 0, -1):
        full = np.kron(full, q[j - 1])
    got = np.array([oracle.kron_element(q, i) for i in range(1 << M)])
    np.testing.assert_allclose(got, full, rtol=1e-14, atol=0)
    # the product state is normalised when every qubit is (norm is multiplicative)
    assert abs(np.linalg.norm(full) - 1) < 1e-13


def test_fused_kron_equals_apply_of_kron_vector():
    M = 11
    gates = wl.random_gates(40, M, 8)
    q = wl.random_qubits(M, 8, "c128")
    full = np.ones(1, dtype=np.complex128)
    for j in range(M, 0, -1):
        full = np.kron(full, q[j - 1])
    ref = oracle.apply_map(oracle.build_map(gates, M), full)
    got = oracle.fused_kron(gates, q)
    np.testing.assert_allclose(got, ref, rtol=1e-14, atol=0)
    part = oracle.fused_kron(gates, q, 300, 77)
    np.testing.assert_array_equal(part, got[300:377])


# ------------------------------------- phased permutations (NEXT(3), R17)
def _all_ext_gates(M):
    gs = list(_all_gates(M))
    for t in range(M):
        gs.append(wl.gate(wl.Z, t))
        for c in range(M):
            if c != t:
                gs.append(wl.gate(wl.CZ, t, c))
                gs.append(wl.gate(wl.SWAP, t, c))
        for c0 in range(M):
            for c1 in range(c0 + 1, M):
                if t not in (c0, c1):
                    gs.append(wl.gate(wl.CCZ, t, c0, c1))
    return gs


def test_paper_matrix_P37_exact_with_phase():
    """Dropping P:L39's "phase gates are not used" admits the P:L37 matrix
    itself, -1 included: the 4-gate circuit of the direction pin followed by
    CZ(a(1), a(2)) reproduces it entry for entry."""
    rows = _rows("example_matrix_P37.txt")
    P = np.zeros((4, 4))
    for r, c, v in rows:
        P[int(r), int(c)] = float(v)
    gates = wl.gates_array([wl.gate(wl.CNOT, 1, 0), wl.gate(wl.NOT, 1),
                            wl.gate(wl.CNOT, 0, 1), wl.gate(wl.NOT, 1), wl.gate(wl.CZ, 0, 1)])
    np.testing.assert_array_equal(dense.composite_matrix(gates, 2), P)
    perm, signs = oracle.build_map_signed(gates, 2)
    assert perm.tolist() == [3, 0, 2, 1]
    assert int(signs[0]) == 0b1000                     # row 3 holds -1
    k1 = wl.make_state(wl.StateSpec(2, "c128", wl.GAUSS, 3))
    np.testing.assert_array_equal(oracle.apply_map_signed(perm, signs, k1), P @ k1)


@pytest.mark.parametrize("M", [2, 3, 4])
def test_ext_step_equals_kronecker_matrix_exhaustive(M):
    for g in _all_ext_gates(M):
        S = dense.step_matrix(g, M)
        assert np.array_equal(S, S.T)                    # symmetric
        cols, vals = dense.signed_perm_of(S)
        assert [oracle.step(g, x) for x in range(1 << M)] == cols.tolist()
        assert [oracle.walk_signed(g, x)[1] for x in range(1 << M)] == vals.astype(int).tolist()
        assert np.array_equal(S @ S, np.eye(1 << M))    # every step is an involution


@pytest.mark.parametrize("M", [2, 3, 4])
def test_ext_composite_equals_dense_product(M):
    for seed in range(30):
        gates = wl.random_gates_ext([0, 1, 3, 8, 15][seed % 5], M, seed,
                                    kinds=(0, 1, 3, 4, 6) if M == 2 else
                                    (0, 1, 2, 3, 4, 5, 6))
        U = dense.composite_matrix(gates, M)
        cols, vals = dense.signed_perm_of(U)
        perm, signs = oracle.build_map_signed(gates, M)
        assert np.array_equal(perm, cols)
        got = np.array([-1.0 if (int(signs[i // 32]) >> (i % 32)) & 1 else 1.0
                        for i in range(1 << M)])
        assert np.array_equal(got, vals)
        k1 = wl.make_state(wl.StateSpec(M, "c128", wl.GAUSS, seed))
        np.testing.assert_array_equal(U @ k1, oracle.apply_map_signed(perm, signs, k1))


@pytest.mark.parametrize("M", [5, 10, 12])
def test_ext_accumulation_equals_composite(M):
    gates = wl.random_gates_ext(60, M, 50 + M)
    for dtype in ("c64", "c128"):
        k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, M))
        perm, signs = oracle.build_map_signed(gates, M)
        want = oracle.apply_map_signed(perm, signs, k1)
        assert oracle.accumulate(gates, k1).tobytes() == want.tobytes()
        assert oracle.run_fused(gates, k1).tobytes() == want.tobytes()


def test_swap_only_is_a_bit_permutation_and_z_only_a_parity():
    M = 10
    rng = np.random.default_rng(2)
    pairs = [tuple(map(int, rng.choice(M, 2, replace=False))) for _ in range(25)]
    gates = wl.gates_array([wl.gate(wl.SWAP, a, b) for a, b in pairs])
    # the composite moves whole bits: bit b of perm[i] is bit src[b] of i,
    # src obtained by applying the swaps in walk order (last gate first)
    src = list(range(M))
    for a, b in reversed(pairs):
        src[a], src[b] = src[b], src[a]
    perm = oracle.build_map(gates, M)
    for i in range(1 << M):
        assert int(perm[i]) == sum(((i >> src[b]) & 1) << b for b in range(M))
    ts = rng.integers(0, M, size=9)
    zg = wl.gates_array([wl.gate(wl.Z, int(t)) for t in ts])
    p2, s2 = oracle.build_map_signed(zg, M)
    assert np.array_equal(p2, np.arange(1 << M, dtype=np.uint32))
    mask = 0
    for t in ts:
        mask ^= 1 << int(t)
    for i in range(1 << M):
        assert ((int(s2[i // 32]) >> (i % 32)) & 1) == bin(i & mask).count("1") % 2


def test_ext_group_identity():
    M = 12
    gates = wl.random_gates_ext(80, M, 9)
    p, s = oracle.build_map_signed(np.concatenate([gates, gates[::-1]]), M)
    assert np.array_equal(p, np.arange(1 << M, dtype=np.uint32)) and not s.any()
