"""GPU parity of the Appendix-1 path (input generated on the fly, fused
with the map) against the oracle.

The GPU forms the Kronecker product with group tables in the state precision
(header qsim.h, qsim_run_fused_kron), the oracle sequentially in double
precision, so the bar is the rounding bound of the arithmetic: a complex
product formed as re = fma(ar, br, -ai*bi), im = fma(ar, bi, ai*br) has
normwise relative error at most 2u (Jeannerod, Kornerup, Louvet & Muller
2017), below the sqrt(5)*u of the plain formula (Brent, Percival &
Zimmermann 2007); the test uses (M-1)*sqrt(5)*u over the M-1 products,
u = 2^-24 (complex64) or 2^-53 (complex128).  Exact special cases (basis
qubits) are compared bit for bit.
"""
import math

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


def tol(M, dtype):
    u = 2.0 ** -24 if dtype == "c64" else 2.0 ** -53
    return 1.01 * max(M - 1, 1) * math.sqrt(5.0) * u


def _check(got, ref, M, dtype):
    err = np.abs(got.astype(np.complex128) - ref)
    bound = tol(M, dtype) * np.abs(ref)
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, (bad[:5], err[bad[:5]], bound[bad[:5]])


def _out(count, dtype):
    return torch.empty(max(count, 1), dtype=torch.complex64 if dtype == "c64" else torch.complex128,
                       device=DEV)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("M", [1, 5, 10, 13, 18])
def test_kron_full(q, M, dtype):
    gates = wl.random_gates(48, M, 3 + M) if M >= 3 else wl.gates_array([wl.gate(wl.NOT, 0)])
    qb = wl.random_qubits(M, 30 + M, dtype)
    ref = oracle.fused_kron(gates, qb)
    walks = [q.WALK_BITSLICED] + ([q.WALK_JIT] if q.jit_status().startswith("ready") else [])
    for walk in walks:
        out = _out(1 << M, dtype)
        q.run_fused_kron(gates, M, qb, out, dtype=dtype, walk=walk)
        torch.cuda.synchronize()
        _check(out.cpu().numpy()[: 1 << M], ref, M, dtype)


@pytest.mark.parametrize("walk", ["bitsliced", "jit"])
def test_kron_ranges(q, walk):
    w = q.WALK_BITSLICED if walk == "bitsliced" else q.WALK_JIT
    if w == q.WALK_JIT and not q.jit_status().startswith("ready"):
        pytest.skip("JIT unavailable")
    M = 15
    gates = wl.random_gates(70, M, 4)
    qb = wl.random_qubits(M, 4, "c64")
    for start, count in ((0, 1), (7, 1000), (1023, 3), (5000, 12000), ((1 << M) - 9, 9), (11, 0)):
        out = _out(count, "c64")
        q.run_fused_kron(gates, M, qb, out, start=start, count=count, dtype="c64", walk=w)
        torch.cuda.synchronize()
        if count:
            _check(out.cpu().numpy()[:count], oracle.fused_kron(gates, qb, start, count), M, "c64")


def test_kron_basis_input_is_exact(q):
    """All qubits |1>: k1 is the basis vector of 2^M - 1, so k2 has
    exactly one 1, at the output whose source is 2^M - 1, zeros elsewhere."""
    M = 16
    gates = wl.random_gates(64, M, 9)
    qb = wl.basis_qubits(M, 1, "c64")
    perm = oracle.build_map(gates, M)
    for walk in (q.WALK_BITSLICED, q.WALK_AUTO):
        out = _out(1 << M, "c64")
        q.run_fused_kron(gates, M, qb, out, dtype="c64", walk=walk)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        want = np.zeros(1 << M, dtype=np.complex64)
        want[int(np.nonzero(perm == (1 << M) - 1)[0][0])] = 1
        assert got.tobytes() == want.tobytes()


@pytest.mark.slow
def test_kron_cfg5_full_size_sampled(q):
    """M = 32, the cfg5 circuit, write-only (no k1 in memory): sampled outputs."""
    cfg = wl.CONFIGS["cfg5"]
    gates, M, N = cfg.gates(), 32, 1 << 32
    qb = wl.random_qubits(M, 2024, "c64")
    out = torch.empty(N, dtype=torch.complex64, device=DEV)
    q.run_fused_kron(gates, M, qb, out, dtype="c64")
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    idx = np.concatenate([[0, 1, 1023, 1024, N - 1], rng.integers(0, N, 4096, dtype=np.uint64)])
    idx = idx.astype(np.uint64)
    src = oracle.walk_many(gates, idx)
    ref = np.array([oracle.kron_element(qb, int(s)) for s in src])
    got = out.index_select(0, torch.from_numpy(idx.astype(np.int64)).to(DEV)).cpu().numpy()
    _check(got, ref, M, "c64")
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("M", [33, 36, 40])
def test_kron_beyond_32_qubits_in_portions(q, M):
    """M > 32: k1 is never stored, so a portion
    [start, start + count) of k2 needs only its own memory ("output in
    convenient continuous portions").  64-bit addresses through the
    NVRTC kernel (64 bit planes) and the per-lane kernel: both within the
    rounding bound of the oracle, equal to each other bit for bit, and
    portions glue (two halves = the whole, byte for byte)."""
    N = 1 << M
    for gates in (wl.random_gates(64, M, 40 + M), wl.random_gates_ext(64, M, 50 + M)):
        qb = wl.random_qubits(M, 60 + M, "c64")
        for start, count in ((0, 1 << 14), (N // 2 - 700, (1 << 15) + 333), (N - 5000, 5000),
                             (0x5a5a5a5a5 % (N - 40000), 40000)):
            ref = oracle.fused_kron(gates, qb, start, count)
            outs = {}
            for w in (q.WALK_JIT, q.WALK_PER_LANE):
                out = _out(count, "c64")
                q.run_fused_kron(gates, M, qb, out, start=start, count=count, dtype="c64", walk=w)
                torch.cuda.synchronize()
                outs[w] = out.cpu().numpy()[:count]
                _check(outs[w], ref, M, "c64")
            assert outs[q.WALK_JIT].tobytes() == outs[q.WALK_PER_LANE].tobytes()
            half = count // 2 + 17
            a, b = _out(half, "c64"), _out(count - half, "c64")
            q.run_fused_kron(gates, M, qb, a, start=start, count=half, dtype="c64")
            q.run_fused_kron(gates, M, qb, b, start=start + half, count=count - half, dtype="c64")
            torch.cuda.synchronize()
            glued = np.concatenate([a.cpu().numpy()[:half], b.cpu().numpy()[:count - half]])
            assert glued.tobytes() == outs[q.WALK_JIT].tobytes()


def test_kron_64bit_kernel_equals_32bit_kernel_below_33(q):
    """For M <= 32 the per-lane 64-bit kernel forms the same products in the
    same order as the 32-bit kernels: identical bytes (c64 and c128)."""
    M = 20
    gates = wl.random_gates_ext(64, M, 77)
    for dtype in ("c64", "c128"):
        qb = wl.random_qubits(M, 8, dtype)
        outs = []
        for w in (q.WALK_PER_LANE, q.WALK_BITSLICED, q.WALK_JIT):
            out = _out(1 << M, dtype)
            q.run_fused_kron(gates, M, qb, out, dtype=dtype, walk=w)
            torch.cuda.synchronize()
            outs.append(out.cpu().numpy().tobytes())
        assert outs[0] == outs[1] == outs[2]


def _kernel_nv(q):
    name = q.last_kernel()
    assert name.startswith("qsim_jit_kron"), name
    return int(name.rsplit("nv ", 1)[1].rstrip(")"))


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("kind", ["random", "structured"])
def test_kron_thread_layout_fast_path(q, dtype, kind):
    """The per-thread hoisted product (qsim_jit.cu kron_source, fast path):
    the host picks 5 output bits whose flips move few source bits; every
    kernel of the call uses the same table layout, so the NVRTC kernel (fast
    path), the per-lane and the bit-sliced kernels give identical bytes, all
    within the rounding bound of the oracle."""
    if not q.jit_status().startswith("ready"):
        pytest.skip("JIT unavailable")
    M = 22
    if kind == "random":    # 64 gates on 22 bits: the sampled |V| is 6..12 by seed
        circuits = [wl.random_gates(64, M, sd) for sd in (122, 126, 127, 120)]
    else:   # gates on bits 0..13 only: bits 14..21 move nothing but themselves
        circuits = [wl.random_gates_ext(96, 14, 5)]
    qb = wl.random_qubits(M, 31, dtype)
    N = 1 << M
    fast = 0
    for gates in circuits:
        outs = {}
        for w in (q.WALK_JIT, q.WALK_PER_LANE, q.WALK_BITSLICED):
            out = _out(N, dtype)
            q.run_fused_kron(gates, M, qb, out, dtype=dtype, walk=w)
            torch.cuda.synchronize()
            if w == q.WALK_JIT:
                fast += _kernel_nv(q) > 0
            outs[w] = out.cpu().numpy()
        assert outs[q.WALK_JIT].tobytes() == outs[q.WALK_PER_LANE].tobytes() == \
            outs[q.WALK_BITSLICED].tobytes()
    assert fast > 0
    _check(outs[q.WALK_JIT], oracle.fused_kron(gates, qb), M, dtype)   # the last circuit, all 2^M


def test_kron_thread_layout_general_path_on_missed_influence(q, monkeypatch):
    """Sampling one point (QSIM_THREAD_BITS_SAMPLES=1) misses most influences: the
    per-warp check then sends tiles down the general path.  Both paths give
    the bytes of the per-lane kernel, with and without phase gates."""
    if not q.jit_status().startswith("ready"):
        pytest.skip("JIT unavailable")
    monkeypatch.setenv("QSIM_THREAD_BITS_SAMPLES", "1")
    M = 22
    for seed in range(6):
        gates = wl.random_gates_ext(48, M, 200 + seed)
        qb = wl.random_qubits(M, seed, "c64")
        a, b = _out(1 << M, "c64"), _out(1 << M, "c64")
        q.run_fused_kron(gates, M, qb, a, dtype="c64", walk=q.WALK_JIT)
        q.run_fused_kron(gates, M, qb, b, dtype="c64", walk=q.WALK_PER_LANE)
        torch.cuda.synchronize()
        assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes(), seed


@pytest.mark.parametrize("start,count", [(0, 1 << 22), (12345, (1 << 22) - 777),
                                         ((1 << 21) - 99, (1 << 22) + 300000), (1 << 22, 1 << 22)])
def test_kron_thread_layout_ranges(q, start, count):
    """Blocks of 2^L outputs hold whole tiles; ranges that cut blocks store
    only their own outputs (bounds checked there): == the per-lane kernel
    byte for byte, within the oracle's bound."""
    if not q.jit_status().startswith("ready"):
        pytest.skip("JIT unavailable")
    M = 23
    gates = wl.random_gates(64, M, 77)
    qb = wl.random_qubits(M, 9, "c64")
    guard = 64
    a = _out(count + guard, "c64")
    a.fill_(7.0)
    b = _out(count, "c64")
    q.run_fused_kron(gates, M, qb, a, start=start, count=count, dtype="c64", walk=q.WALK_JIT)
    q.run_fused_kron(gates, M, qb, b, start=start, count=count, dtype="c64", walk=q.WALK_PER_LANE)
    torch.cuda.synchronize()
    ga = a.cpu().numpy()
    assert ga[:count].tobytes() == b.cpu().numpy()[:count].tobytes()
    assert np.all(ga[count:] == 7.0)        # nothing written past the range
    sel = np.unique(np.concatenate([np.arange(min(count, 2000)), np.arange(count - min(count, 2000), count)]))
    _check(ga[sel], oracle.fused_kron(gates, qb, start, count)[sel], M, "c64")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_kron_thread_layout_beyond_32_qubits_ragged(q, dtype):
    """M = 36, a 2^22 + 12345-entry portion at an unaligned start: 64-bit
    planes, the in-thread layout with blocks of 2^L cut at both ends; the
    NVRTC kernel == the per-lane 64-bit kernel byte for byte, within the
    oracle's rounding bound on sampled outputs, nothing written past the end."""
    if not q.jit_status().startswith("ready"):
        pytest.skip("JIT unavailable")
    M = 36
    gates = wl.random_gates(64, M, 36)
    qb = wl.random_qubits(M, 11, dtype)
    start, count = (1 << 35) - 987654, (1 << 22) + 12345
    guard = 32
    a = _out(count + guard, dtype)
    a.fill_(3.0)
    b = _out(count, dtype)
    q.run_fused_kron(gates, M, qb, a, start=start, count=count, dtype=dtype, walk=q.WALK_JIT)
    name = q.last_kernel()
    q.run_fused_kron(gates, M, qb, b, start=start, count=count, dtype=dtype, walk=q.WALK_PER_LANE)
    torch.cuda.synchronize()
    ga = a.cpu().numpy()
    assert name.startswith("qsim_jit_kron"), name
    assert ga[:count].tobytes() == b.cpu().numpy()[:count].tobytes()
    assert np.all(ga[count:] == 3.0)
    for s0, c0 in ((0, 3000), (count // 2, 3000), (count - 3000, 3000)):
        _check(ga[s0:s0 + c0], oracle.fused_kron(gates, qb, start + s0, c0), M, dtype)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_kron_at_63_qubits(q, dtype):
    """The largest M the 64-bit walk takes (M = 63): portions at both ends and
    in the middle, and a 2^22 + 77 portion ending at the last output (the
    in-thread layout with cut blocks), NVRTC == per-lane kernel byte for byte,
    within the oracle's bound."""
    if not q.jit_status().startswith("ready"):
        pytest.skip("JIT unavailable")
    M = 63
    N = 1 << M
    gates = wl.random_gates_ext(96, M, 63)
    qb = wl.random_qubits(M, 17, dtype)
    for start, count in ((0, 5000), (N - 5000, 5000), ((1 << 62) + 12345, 7777),
                         (N - (1 << 22) - 77, (1 << 22) + 77)):
        outs = {}
        for w in (q.WALK_JIT, q.WALK_PER_LANE):
            out = _out(count, dtype)
            q.run_fused_kron(gates, M, qb, out, start=start, count=count, dtype=dtype, walk=w)
            torch.cuda.synchronize()
            outs[w] = out.cpu().numpy()[:count]
        assert outs[q.WALK_JIT].tobytes() == outs[q.WALK_PER_LANE].tobytes(), (start, count)
        for s0 in sorted({0, max(count - 3000, 0)}):
            c0 = min(3000, count - s0)
            _check(outs[q.WALK_JIT][s0:s0 + c0], oracle.fused_kron(gates, qb, start + s0, c0), M, dtype)


@pytest.mark.slow
def test_kron_c128_full_size_sampled(q):
    """complex128 at M = 32: 2^32 outputs, 64 GiB written without any input
    in memory; sampled outputs within the oracle's bound."""
    M, N = 32, 1 << 32
    gates = wl.CONFIGS["cfg5"].gates()
    qb = wl.random_qubits(M, 2025, "c128")
    out = torch.empty(N, dtype=torch.complex128, device=DEV)
    q.run_fused_kron(gates, M, qb, out, dtype="c128")
    torch.cuda.synchronize()
    rng = np.random.default_rng(2)
    idx = np.concatenate([[0, 1, N - 1], rng.integers(0, N, 3000, dtype=np.uint64)]).astype(np.uint64)
    src = oracle.walk_many(gates, idx)
    ref = np.array([oracle.kron_element(qb, int(s)) for s in src])
    got = out.index_select(0, torch.from_numpy(idx.astype(np.int64)).to(DEV)).cpu().numpy()
    _check(got, ref, M, "c128")
    del out
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_kron_portions_glue_at_32_qubits(q, dtype):
    """The table grouping is the circuit's, not the range's: at
    M = 32 the whole output in one call equals, byte for byte, portions
    computed by separate calls below 2^22 outputs (ahead-of-time kernels),
    above it (NVRTC, in-thread layout), misaligned and ragged -- and a
    sampled set of outputs lies within the oracle's rounding bound."""
    M, N = 32, 1 << 32
    gates = wl.CONFIGS["cfg5"].gates()
    qb = wl.random_qubits(M, 2024, dtype)
    e = 8 if dtype == "c64" else 16
    if dtype == "c128":              # 64 GiB: check the upper half as "the whole" range instead
        whole_start, whole_count = N // 2, N // 2
    else:
        whole_start, whole_count = 0, N
    whole = torch.empty(whole_count * e, dtype=torch.uint8, device=DEV)
    q.run_fused_kron(gates, M, qb, whole, start=whole_start, count=whole_count, dtype=dtype)
    torch.cuda.synchronize()
    portions = [(whole_start, 1 << 21), (whole_start + (1 << 30) - 12345, (1 << 23) + 77),
                (whole_start + whole_count - (1 << 22) - 5, (1 << 22) + 5),
                (whole_start + (1 << 28), 1 << 26), (whole_start + 3, 1000)]
    for start, count in portions:
        part = torch.empty(count * e, dtype=torch.uint8, device=DEV)
        q.run_fused_kron(gates, M, qb, part, start=start, count=count, dtype=dtype)
        torch.cuda.synchronize()
        off = (start - whole_start) * e
        assert torch.equal(part, whole[off:off + count * e]), (start, count, q.last_kernel())
    rng = np.random.default_rng(3)
    idx = np.unique(rng.integers(whole_start, whole_start + whole_count, 2000, dtype=np.uint64))
    ref = np.array([oracle.fused_kron(gates, qb, int(i), 1)[0] for i in idx])
    got = whole.view(-1, e)[torch.from_numpy((idx - whole_start).astype(np.int64)).to(DEV)]
    got = got.cpu().numpy().reshape(-1).view(wl.NP_DTYPE[dtype])
    _check(got, ref, M, dtype)
    del whole
    torch.cuda.empty_cache()
