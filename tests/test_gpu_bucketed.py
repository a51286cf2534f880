"""GPU parity of the two-pass cluster-bucketed path (qsim_run_bucketed;
well-mixed circuits such as cfg3): every output against the oracle, byte for
byte (readings R1/R2/R15), with and without the stored map, complex64
and complex128, phase / SWAP circuits (R17), bucket counts from 1 to 512, and
the argument checks of the C ABI."""
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


@pytest.mark.parametrize("dtype,M", [("c64", 18), ("c128", 17), ("c64", 21), ("c128", 20),
                                     ("c64", 24), ("c128", 24), ("c64", 26)])
@pytest.mark.parametrize("with_perm", [False, True])
def test_bucketed_equals_oracle(q, M, dtype, with_perm):
    gates = wl.random_gates(160, M, 900 + M)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 90 + M))
    perm_ref = oracle.build_map(gates, M)
    ref = oracle.apply_map(perm_ref, k1)
    k1_d = _dev(k1)
    k2_d = torch.full_like(k1_d, 0xA5)
    nb = q.bucket_scratch_bytes(M, dtype, with_perm)
    assert nb > 0
    scratch = torch.empty(nb, dtype=torch.uint8, device=DEV)
    perm = torch.full((1 << M,), -1, dtype=torch.int32, device=DEV) if with_perm else None
    for _ in range(2):                       # repeated calls (cursor reset, kernel cache)
        q.run_bucketed(gates, M, k1_d, k2_d, scratch, perm_out=perm, dtype=dtype)
        torch.cuda.synchronize()
        assert k2_d.cpu().numpy().tobytes() == ref.tobytes()
        if with_perm:
            assert np.array_equal(perm.cpu().numpy().view(np.uint32), perm_ref)
    if q.jit_status().startswith("ready"):
        assert q.last_kernel().startswith("qsim_bucket_pass1")


@pytest.mark.parametrize("M", [18, 22])
def test_bucketed_phase_and_swap_circuits(q, M):
    gates = wl.random_gates_ext(120, M, 31 + M)
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 3 + M))
    perm, signs = oracle.build_map_signed(gates, M)
    ref = oracle.apply_map_signed(perm, signs, k1)
    k1_d = _dev(k1)
    k2_d = torch.empty_like(k1_d)
    scratch = torch.empty(q.bucket_scratch_bytes(M, "c64"), dtype=torch.uint8, device=DEV)
    q.run_bucketed(gates, M, k1_d, k2_d, scratch, dtype="c64")
    torch.cuda.synchronize()
    assert k2_d.cpu().numpy().tobytes() == ref.tobytes()
    pm = torch.empty(1 << M, dtype=torch.int32, device=DEV)
    big = torch.empty(q.bucket_scratch_bytes(M, "c64", True), dtype=torch.uint8, device=DEV)
    with pytest.raises(q.QsimError) as ei:          # a uint32 map cannot hold -1 rows
        q.run_bucketed(gates, M, k1_d, k2_d, big, perm_out=pm, dtype="c64")
    assert ei.value.code == q.EINVAL


def test_bucketed_argument_checks(q):
    M = 19
    gates = wl.random_gates(40, M, 1)
    k1 = torch.zeros((1 << M) * 8, dtype=torch.uint8, device=DEV)
    k2 = torch.empty_like(k1)
    nb = q.bucket_scratch_bytes(M, "c64")
    scratch = torch.empty(nb, dtype=torch.uint8, device=DEV)
    with pytest.raises(q.QsimError) as ei:                      # scratch too small
        q.run_bucketed(gates, M, k1, k2, scratch[:nb - 16], dtype="c64")
    assert ei.value.code == q.EINVAL
    with pytest.raises(q.QsimError) as ei:                      # scratch overlaps k2
        q.run_bucketed(gates, M, k1, k2, k2, dtype="c64")
    assert ei.value.code in (q.EALIAS, q.EINVAL)
    with pytest.raises(q.QsimError) as ei:                      # M below one bucket
        q.run_bucketed(wl.random_gates(10, 12, 1), 12, k1, k2, scratch, dtype="c64")
    assert ei.value.code == q.ERANGE
    assert q.bucket_scratch_bytes(32, "c64") == 0               # > 512 buckets
    assert q.bucket_scratch_bytes(12, "c64") == 0
    assert q.bucket_scratch_bytes(26, "c128") > 0 and q.bucket_scratch_bytes(28, "c128") == 0
