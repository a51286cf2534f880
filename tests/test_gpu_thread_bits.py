"""GPU parity of the in-thread output bits (qsim_api.cu thread_bits; the
NVRTC build and on-the-fly input kernels): a thread's 32 outputs differ in 5
output bits J chosen so that their sources differ in few address bits V;
the build's fast path takes the 32 sources as one source XOR combinations
of 5 difference columns (when V's planes are affine in J, checked per warp).  The map is integer
work: bit-exact against the oracle, with J at any position,
ragged ranges, and tiles where a sampled-away influence sends the warp down
the general path."""
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
    if not q.jit_status().startswith("ready"):
        pytest.skip("JIT unavailable")
    return q


def _nv(name):
    return int(name.rsplit("nv ", 1)[1].rstrip(")"))


def _build(q, gates, M, start, count, guard=0):
    out = torch.from_numpy(np.full(count + guard, 0xABCDEF01, dtype=np.uint32).view(np.int32)).to(DEV)
    q.build_map_range(gates, M, start, count, out, walk=q.WALK_JIT)
    torch.cuda.synchronize()
    name = q.last_kernel()
    return out.cpu().numpy().view(np.uint32), name


@pytest.mark.parametrize("kind", ["random", "structured", "swaps"])
def test_build_thread_bits_full(q, kind):
    M = 22
    if kind == "random":
        circuits = [wl.random_gates(64, M, sd) for sd in (122, 126, 127, 120, 3)]
    elif kind == "structured":      # bits 14..21 never move
        circuits = [wl.random_gates(96, 14, 5)]
    else:                           # SWAP renaming + NOT/CNOT/CCNOT (on bits 0..15, and on all)
        kinds = (wl.NOT, wl.CNOT, wl.CCNOT, wl.SWAP)
        circuits = [wl.random_gates_ext(64, 16, 9, kinds=kinds), wl.random_gates_ext(64, M, 9, kinds=kinds)]
    fast = 0
    for gates in circuits:
        got, name = _build(q, gates, M, 0, 1 << M)
        assert name.startswith("qsim_jit_build"), name
        fast += _nv(name) > 0
        assert np.array_equal(got, oracle.build_map(gates, M))
    assert fast > 0


@pytest.mark.parametrize("start,count", [(0, 1 << 22), (12345, (1 << 22) - 777),
                                         ((1 << 21) - 99, (1 << 22) + 300000), (1 << 22, 1 << 22)])
def test_build_thread_bits_ranges(q, start, count):
    """Blocks of 2^L outputs hold whole tiles; a range that cuts blocks
    stores only its own outputs, nothing past the end."""
    M = 23
    gates = wl.random_gates(64, M, 77)
    got, name = _build(q, gates, M, start, count, guard=64)
    assert np.array_equal(got[:count], oracle.build_map(gates, M, start, count))
    assert np.all(got[count:] == 0xABCDEF01)


def test_build_thread_bits_general_path_on_missed_influence(q, monkeypatch):
    """One sample point misses most influences: the per-warp check sends
    tiles down the general path; the map stays exact."""
    monkeypatch.setenv("QSIM_THREAD_BITS_SAMPLES", "1")
    M = 22
    for seed in range(6):
        gates = wl.random_gates(48, M, 300 + seed)
        got, _ = _build(q, gates, M, 0, 1 << M)
        assert np.array_equal(got, oracle.build_map(gates, M)), seed


def test_build_thread_bits_off_equals_on(q, monkeypatch):
    """QSIM_THREAD_BITS=0 (J = 5..9, no fast path) gives the same map."""
    M = 24
    gates = wl.random_gates(64, M, 11)
    on, name_on = _build(q, gates, M, 0, 1 << M)
    monkeypatch.setenv("QSIM_THREAD_BITS", "0")
    off, name_off = _build(q, gates, M, 0, 1 << M)
    monkeypatch.setenv("QSIM_THREAD_BITS", "1")
    monkeypatch.setenv("QSIM_BUILD_THREAD_BITS", "0")
    plain, name_plain = _build(q, gates, M, 0, 1 << M)
    assert "J 5.6.7.8.9" in name_plain
    assert np.array_equal(on, plain)
    assert "J 5.6.7.8.9" in name_off and _nv(name_off) == 0
    assert np.array_equal(on, off)


def test_thread_bits_long_circuit_on_quiet_bits(q):
    """1500 gates (> 1024: the host samples 16 points and 4 warps) on bits
    0..15 of M = 23: bits 16..22 are quiet, so both kernels take their fast
    paths.  The map equals the ahead-of-time per-lane walk byte for byte and
    the oracle on sampled outputs; the on-the-fly input equals the per-lane
    kernel byte for byte."""
    M = 23
    gates = wl.random_gates(1500, 16, 21)
    got, name = _build(q, gates, M, 0, 1 << M)
    assert _nv(name) > 0, name
    ref = torch.empty(1 << M, dtype=torch.int32, device=DEV)
    q.build_map_range(gates, M, 0, 1 << M, ref, walk=q.WALK_PER_LANE)
    torch.cuda.synchronize()
    assert np.array_equal(got, ref.cpu().numpy().view(np.uint32))
    rng = np.random.default_rng(5)
    idx = np.concatenate([np.arange(64), rng.integers(0, 1 << M, 3000), np.arange((1 << M) - 64, 1 << M)])
    assert np.array_equal(got[idx], oracle.walk_many(gates, idx.astype(np.uint64)))
    qb = wl.random_qubits(M, 3, "c64")
    a = torch.empty(1 << M, dtype=torch.complex64, device=DEV)
    b = torch.empty_like(a)
    q.run_fused_kron(gates, M, qb, a, dtype="c64", walk=q.WALK_JIT)
    kname = q.last_kernel()
    q.run_fused_kron(gates, M, qb, b, dtype="c64", walk=q.WALK_PER_LANE)
    torch.cuda.synchronize()
    assert _nv(kname) > 0, kname
    assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes()
