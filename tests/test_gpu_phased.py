"""GPU parity for phased permutations (reading R17): Z, CZ,
CCZ (rows with value -1) and SWAP steps, through every call that accepts them,
against the oracle byte for byte (-1 is an IEEE negation of both parts, done
on the sign bits on both sides)."""
import numpy as np
import pytest

import oracle
import workloads as wl

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def q():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_native()
    import paper_quant_ph_0308158_b200 as q
    return q


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).to(DEV)


def _signed_ref(gates, M, k1, start=0, count=None):
    perm, signs = oracle.build_map_signed(gates, M, start, count)
    return perm, signs, oracle.apply_map_signed(perm, signs, k1)


def test_paper_matrix_P37_on_the_gpu(q):
    """The P:L37 matrix, -1 included (the oracle pin's circuit): its columns
    come out of run_fused applied to the basis vectors."""
    gates = wl.gates_array([wl.gate(wl.CNOT, 1, 0), wl.gate(wl.NOT, 1), wl.gate(wl.CNOT, 0, 1),
                            wl.gate(wl.NOT, 1), wl.gate(wl.CZ, 0, 1)])
    P = np.zeros((4, 4), dtype=np.complex128)
    P[0, 3], P[1, 0], P[2, 2], P[3, 1] = 1, 1, 1, -1
    for j in range(4):
        e = np.zeros(4, dtype=np.complex128)
        e[j] = 1.0
        k2 = torch.empty(64, dtype=torch.uint8, device=DEV)
        q.run_fused(gates, 2, _dev(e), k2, dtype="c128")
        torch.cuda.synchronize()
        np.testing.assert_array_equal(k2.cpu().numpy().view(np.complex128), P[:, j])


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("M", [3, 9, 13, 17])
def test_fused_all_walks(q, M, dtype):
    gates = wl.random_gates_ext(90, M, 700 + M)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 5 + M))
    _, _, ref = _signed_ref(gates, M, k1)
    assert ref.tobytes() == oracle.accumulate(gates, k1).tobytes()   # two oracles agree
    k1_d = _dev(k1)
    N = 1 << M
    for walk in (q.WALK_AUTO, q.WALK_PER_LANE, q.WALK_BITSLICED):
        out = torch.empty_like(k1_d)
        q.run_fused_range(gates, M, 0, N, k1_d, out, dtype=dtype, walk=walk)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == ref.tobytes(), walk
    # ragged range
    s, c = (N // 3) | 1, N // 2 + 5 if N > 8 else 3
    e = 8 if dtype == "c64" else 16
    out = torch.empty(c * e, dtype=torch.uint8, device=DEV)
    q.run_fused_range(gates, M, s, c, k1_d, out, dtype=dtype, walk=q.WALK_BITSLICED)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == ref[s:s + c].tobytes()


@pytest.mark.parametrize("M", [5, 12, 16])
def test_build_and_apply_signed(q, M):
    gates = wl.random_gates_ext(70, M, 800 + M)
    N = 1 << M
    cases = [(0, N), (32, N - 32 - 7), (N - 32, 13), (64, 0)]
    for start, count in [(s0, c0) for s0, c0 in cases if c0 >= 0 and s0 + c0 <= N]:
        perm_ref, signs_ref = oracle.build_map_signed(gates, M, start, count)
        perm = torch.empty(max(count, 1), dtype=torch.int32, device=DEV)
        signs = torch.full((max((count + 31) // 32, 1),), -1, dtype=torch.int32, device=DEV)
        q.build_map_signed(gates, M, start, count, perm, signs)
        torch.cuda.synchronize()
        if count:
            assert np.array_equal(perm.cpu().numpy().view(np.uint32)[:count], perm_ref)
            assert np.array_equal(signs.cpu().numpy().view(np.uint32)[:(count + 31) // 32],
                                  signs_ref[:(count + 31) // 32]), (start, count)
    for dtype in ("c64", "c128"):
        k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, M))
        perm_ref, signs_ref, ref = _signed_ref(gates, M, k1)
        perm = torch.from_numpy(perm_ref.view(np.int32)).to(DEV)
        signs = torch.from_numpy(signs_ref.view(np.int32)).to(DEV)
        k1_d = _dev(k1)
        for count in (N, N - 3):
            out = torch.empty_like(k1_d)
            q.apply_map_signed(perm, signs, count, M, k1_d, out, dtype=dtype)
            torch.cuda.synchronize()
            e = 8 if dtype == "c64" else 16
            assert out.cpu().numpy()[:count * e].tobytes() == ref[:count].tobytes()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("M", [12, 17])
def test_planned_fused_signed(q, M, dtype):
    """run_fused_planned (NVRTC kernel with the sign in registers, and the
    ahead-of-time kernel without a workspace) in the plan's order."""
    gates = wl.random_gates_ext(80, M, 900 + M)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 2 * M))
    _, _, ref = _signed_ref(gates, M, k1)
    k1_d = _dev(k1)
    plan = q.plan_create(gates, M, dtype)
    plan.flags = 0
    for w in (q.workspace(), None):
        out = torch.empty_like(k1_d)
        q.run_fused_planned(plan, gates, k1_d, out, w)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == ref.tobytes(), w is None


def test_kron_with_phases_is_the_signed_plain_result(q):
    """Input on the fly (Appendix 1) with phase steps: the phase steps move no
    address, so k2 equals the result of the circuit without them, negated
    exactly on the rows the oracle marks -1 (JIT and bit-sliced walks)."""
    M = 14
    gates = wl.random_gates_ext(60, M, 31)
    plain = np.ascontiguousarray(gates[(gates[:, 0] < 3) | (gates[:, 0] == 6)])
    rng = np.random.default_rng(4)
    qubits = (rng.normal(size=(M, 2)) + 1j * rng.normal(size=(M, 2))).astype(np.complex128)
    _, signs = oracle.build_map_signed(gates, M)
    neg = np.array([(int(signs[i // 32]) >> (i % 32)) & 1 for i in range(1 << M)], dtype=bool)
    for dtype, e in (("c64", 8), ("c128", 16)):
        for walk in (q.WALK_BITSLICED, q.WALK_JIT):
            a = torch.empty((1 << M) * e, dtype=torch.uint8, device=DEV)
            b = torch.empty_like(a)
            q.run_fused_kron(gates, M, qubits, a, dtype=dtype, walk=walk)
            q.run_fused_kron(plain, M, qubits, b, dtype=dtype, walk=walk)
            torch.cuda.synchronize()
            na = a.cpu().numpy().view(np.complex64 if e == 8 else np.complex128)
            nb = b.cpu().numpy().view(np.complex64 if e == 8 else np.complex128)
            want = np.where(neg, -nb, nb)
            assert na.tobytes() == want.tobytes(), (dtype, walk)


def test_swap_circuits_through_the_unsigned_calls(q):
    """SWAP is a plain permutation: build_map (JIT and interpreter), apply,
    and the planned one-pass map + gather accept it."""
    M = 16
    rng = np.random.default_rng(7)
    gates = wl.random_gates_ext(70, M, 12, kinds=(wl.NOT, wl.CNOT, wl.CCNOT, wl.SWAP))
    assert (gates[:, 0] == wl.SWAP).any()
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 1))
    perm_ref = oracle.build_map(gates, M)
    ref = oracle.apply_map(perm_ref, k1)
    k1_d = _dev(k1)
    for walk in (q.WALK_PER_LANE, q.WALK_BITSLICED, q.WALK_JIT):
        perm = torch.empty(1 << M, dtype=torch.int32, device=DEV)
        q.build_map_range(gates, M, 0, 1 << M, perm, walk=walk)
        torch.cuda.synchronize()
        assert np.array_equal(perm.cpu().numpy().view(np.uint32), perm_ref), walk
    out = torch.empty_like(k1_d)
    q.apply_map(perm, M, k1_d, out, dtype="c64")
    plan = q.plan_create(gates, M, "c64")
    plan.flags = 0
    pm = torch.empty_like(perm)
    out2 = torch.empty_like(k1_d)
    q.map_gather_planned(plan, gates, pm, k1_d, out2, q.workspace())
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == ref.tobytes()
    assert out2.cpu().numpy().tobytes() == ref.tobytes()
    assert np.array_equal(pm.cpu().numpy().view(np.uint32), perm_ref)
    del rng
