"""GPU parity: the CUDA path through the C ABI against the CPU oracle.

Bit-exact throughout (pure index arithmetic and data movement; DESIGN.md
"Parity bar").  Entries are compared as raw bytes / integer views, never as
floats (R15).

* small and medium sizes: every output compared with the oracle, both walk
  algorithms, complex64 and complex128, ragged ranges, edge cases;
* BASELINE.json configs: cfg1/cfg2 in full here; cfg3/cfg4/cfg5 every output
  at full size in tests/test_gpu_fullsize.py, plus the index-tagged M = 32
  gather below.
"""
import numpy as np
import pytest

import oracle
import workloads as wl

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_native()
    import paper_quant_ph_0308158_b200 as q
    return q


DEV = "cuda:0"
WALKS = [1, 2]   # WALK_PER_LANE, WALK_BITSLICED


def _to_dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).to(DEV)


def _perm_np(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def _new_perm(count):
    return torch.empty(max(count, 1), dtype=torch.int32, device=DEV)


def _new_state(count, dtype):
    return torch.empty(max(count, 1) * (8 if dtype == "c64" else 16), dtype=torch.uint8,
                       device=DEV)


# ------------------------------------------------------------- full compares
@pytest.mark.parametrize("M", [1, 2, 3, 5, 9, 10, 11, 13, 16])
@pytest.mark.parametrize("walk", WALKS)
def test_build_full_small(q, M, walk):
    for seed, n in ((M, 0), (M + 1, 1), (M + 2, 37), (M + 3, 300)):
        if M >= 3:
            gates = wl.random_gates(n, M, seed)
        else:
            gates = wl.gates_array([wl.gate(wl.NOT, s % M) if M == 1 or s % 2
                                    else wl.gate(wl.CNOT, s % 2, 1 - s % 2) for s in range(n)])
        N = 1 << M
        perm = _new_perm(N)
        q.build_map_range(gates, M, 0, N, perm, walk=walk)
        torch.cuda.synchronize()
        assert np.array_equal(_perm_np(perm)[:N], oracle.build_map(gates, M)), (M, n, walk)


@pytest.mark.parametrize("M", [3, 10, 16, 23])
def test_build_jit(q, M):
    """Circuit-specialised (NVRTC) build kernel: full compare, ragged ranges."""
    if not q.jit_status().startswith("ready"):
        pytest.skip(f"JIT unavailable: {q.jit_status()}")
    N = 1 << M
    for seed, n in ((M, 0), (M + 1, 1), (M + 2, 64), (M + 3, 257)):
        gates = wl.random_gates(n, M, seed)
        want = oracle.build_map(gates, M)
        perm = _new_perm(N)
        q.build_map_range(gates, M, 0, N, perm, walk=q.WALK_JIT)
        torch.cuda.synchronize()
        assert np.array_equal(_perm_np(perm)[:N], want), (M, n)
        for start, count in ((5, min(N - 5, 3000)), (N - 3, 3), (N // 2, N // 2)):
            pr = _new_perm(count)
            q.build_map_range(gates, M, start, count, pr, walk=q.WALK_JIT)
            torch.cuda.synchronize()
            assert np.array_equal(_perm_np(pr)[:count], want[start:start + count])
    rg = wl.ripple_gates(M, 200) if M >= 3 else None
    if rg is not None:
        perm = _new_perm(N)
        q.build_map_range(rg, M, 0, N, perm, walk=q.WALK_JIT)
        torch.cuda.synchronize()
        assert np.array_equal(_perm_np(perm)[:N], oracle.build_map(rg, M))


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("M", [4, 12, 17])
def test_apply_and_fused_full(q, M, dtype):
    gates = wl.random_gates(64, M, 10 + M)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, M))
    ref = oracle.apply_map(oracle.build_map(gates, M), k1)
    k1_d = _to_dev(k1)
    perm = _new_perm(1 << M)
    q.build_map(gates, M, perm)
    k2 = torch.empty_like(k1_d)
    q.apply_map(perm, M, k1_d, k2, dtype=dtype)
    torch.cuda.synchronize()
    assert k2.cpu().numpy().tobytes() == ref.tobytes()
    for walk in WALKS:
        k2f = torch.empty_like(k1_d)
        q.run_fused_range(gates, M, 0, 1 << M, k1_d, k2f, dtype=dtype, walk=walk)
        torch.cuda.synchronize()
        assert k2f.cpu().numpy().tobytes() == ref.tobytes(), walk


@pytest.mark.parametrize("walk", WALKS)
def test_ragged_ranges(q, walk):
    """Continuous portions with starts/ends off the 1024-entry tiles."""
    M = 15
    gates = wl.random_gates(90, M, 3)
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 4))
    k1_d = _to_dev(k1)
    perm_all = oracle.build_map(gates, M)
    for start, count in ((0, 1), (1, 1), (5, 1023), (1023, 2), (1000, 3000), (4096, 4096),
                         ((1 << M) - 7, 7), (123, 0), (0, 1 << M)):
        pr = _new_perm(count)
        q.build_map_range(gates, M, start, count, pr, walk=walk)
        k2r = _new_state(count, "c64")
        q.run_fused_range(gates, M, start, count, k1_d, k2r, dtype="c64", walk=walk)
        torch.cuda.synchronize()
        assert np.array_equal(_perm_np(pr)[:count], perm_all[start:start + count])
        want = oracle.run_fused(gates, k1, start, count)
        assert k2r.cpu().numpy()[:count * 8].tobytes() == want.tobytes()


def test_apply_ragged_counts(q):
    M = 12
    k1 = wl.make_state(wl.StateSpec(M, "c128", wl.GAUSS, 8))
    k1_d = _to_dev(k1)
    perm = oracle.build_map(wl.random_gates(50, M, 8), M)
    for count in (0, 1, 3, 4, 5, 1021, 4096):
        p_d = torch.from_numpy(perm[:max(count, 1)].view(np.int32).copy()).to(DEV)
        k2 = _new_state(count, "c128")
        q.apply_map_range(p_d, count, M, k1_d, k2, dtype="c128")
        torch.cuda.synchronize()
        assert k2.cpu().numpy()[:count * 16].tobytes() == oracle.apply_map(perm[:count], k1).tobytes()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("M", [10, 11, 14, 17])
def test_planned_apply_and_fused(q, M, dtype):
    """sigma-ordered traversal (plans): same bytes as the oracle for every
    chunk size / occupancy / scheduling variant."""
    gates = wl.random_gates(80, M, 70 + M)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 7 + M))
    ref = oracle.apply_map(oracle.build_map(gates, M), k1)
    k1_d = _to_dev(k1)
    perm = _new_perm(1 << M)
    q.build_map(gates, M, perm)
    plan = q.plan_create(gates, M, dtype)
    assert sorted(list(plan.sigma)[:M]) == list(range(M))
    if M >= 17:                                          # beyond the sector cover + runs
        assert list(plan.sigma)[:M] != list(range(M))   # a real reordering
    plan.flags = 0                                       # force the sigma kernels
    ws = q.workspace()
    for cl in sorted({10, min(M, 12), M}):
        for bps, thr in ((1, 256), (2, 256), (8, 256), (1, 512)):   # 512: 16-warp NVRTC kernels
            for w in (ws, None):
                plan.chunk_log2, plan.blocks_per_sm, plan.fused_chunk_log2 = cl, bps, cl
                plan.cta_threads = thr
                out = torch.empty_like(k1_d)
                q.apply_map_planned(plan, perm, k1_d, out, w)
                outf = torch.empty_like(k1_d)
                q.run_fused_planned(plan, gates, k1_d, outf, w)
                outm = torch.empty_like(k1_d)
                pm = _new_perm(1 << M)
                q.map_gather_planned(plan, gates, pm, k1_d, outm, w)
                torch.cuda.synchronize()
                assert out.cpu().numpy().tobytes() == ref.tobytes(), (cl, bps, thr)
                assert outf.cpu().numpy().tobytes() == ref.tobytes(), (cl, bps, thr)
                assert outm.cpu().numpy().tobytes() == ref.tobytes(), (cl, bps, thr)
                assert np.array_equal(_perm_np(pm), _perm_np(perm)), (cl, bps, thr)
                # the two-kernel map + gather (planned gather, natural-order build)
                sp = q.Plan.from_buffer_copy(plan)
                sp.flags |= q.PLAN_SPLIT
                outs, ps = torch.empty_like(k1_d), _new_perm(1 << M)
                q.map_gather_planned(sp, gates, ps, k1_d, outs, w)
                torch.cuda.synchronize()
                assert outs.cpu().numpy().tobytes() == ref.tobytes(), ("split", cl, bps, thr)
                assert np.array_equal(_perm_np(ps), _perm_np(perm)), ("split", cl, bps, thr)


@pytest.mark.parametrize("dtype,M", [("c64", 12), ("c64", 14), ("c64", 17), ("c128", 11),
                                     ("c128", 15)])
def test_planned_orders_moving_lane_bits(q, M, dtype):
    """Traversal orders whose lane bits are not output bits 3..4 (the sector
    cover puts other bits there; only 0..2 / 0..1 are kept): the plan's own
    sigma and a sigma reversing every non-kept bit, through the NVRTC kernels
    with the chunk ticket (workspace) and with round-robin chunks (no
    workspace) -- same bytes."""
    gates = wl.random_gates(80, M, 300 + M)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 11 + M))
    perm_ref = oracle.build_map(gates, M)
    ref = oracle.apply_map(perm_ref, k1)
    k1_d = _to_dev(k1)
    perm = _new_perm(1 << M)
    q.build_map(gates, M, perm)
    keep = 3 if dtype == "c64" else 2
    plan = q.plan_create(gates, M, dtype)
    plan.flags = 0
    sigmas = [list(plan.sigma)[:M], list(range(keep)) + list(range(M - 1, keep - 1, -1))]
    for sig in sigmas:
        for k, b in enumerate(sig):
            plan.sigma[k] = b
        for w in (q.workspace(), None):
            out, outf, outm = (torch.empty_like(k1_d) for _ in range(3))
            pm = _new_perm(1 << M)
            q.apply_map_planned(plan, perm, k1_d, out, w)
            q.run_fused_planned(plan, gates, k1_d, outf, w)
            q.map_gather_planned(plan, gates, pm, k1_d, outm, w)
            torch.cuda.synchronize()
            for o in (out, outf, outm):
                assert o.cpu().numpy().tobytes() == ref.tobytes(), (sig, w is None)
            assert np.array_equal(_perm_np(pm), perm_ref)


@pytest.mark.parametrize("dtype,M,ext", [("c64", 13, False), ("c64", 18, False), ("c128", 16, False),
                                         ("c64", 17, True)])
def test_plain_run_fused_is_planned(q, M, dtype, ext):
    """qsim_run_fused over the whole output plans internally (plan cached per
    circuit) and runs the NVRTC kernel in the plan's order: same bytes as
    the oracle, also for phase / SWAP circuits (R17) and on repeated calls."""
    gates = (wl.random_gates_ext(70, M, 40 + M) if ext else wl.random_gates(70, M, 40 + M))
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 5 + M))
    if ext:
        perm, signs = oracle.build_map_signed(gates, M)
        ref = oracle.apply_map_signed(perm, signs, k1)
    else:
        ref = oracle.apply_map(oracle.build_map(gates, M), k1)
    k1_d = _to_dev(k1)
    for _ in range(2):
        out = torch.empty_like(k1_d)
        q.run_fused(gates, M, k1_d, out, dtype=dtype)
        torch.cuda.synchronize()
        if q.jit_status().startswith("ready"):
            assert q.last_kernel() in ("qsim_jit_fused", "qsim_jit_local"), q.last_kernel()
        assert out.cpu().numpy().tobytes() == ref.tobytes()


def test_planned_small_M_falls_back_to_natural(q):
    for M in (1, 3, 9):
        gates = wl.random_gates(20, M, M) if M >= 3 else wl.gates_array([wl.gate(wl.NOT, 0)])
        k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 1))
        ref = oracle.apply_map(oracle.build_map(gates, M), k1)
        plan = q.plan_create(gates, M, "c64")
        k1_d = _to_dev(k1)
        perm = _new_perm(1 << M)
        q.build_map(gates, M, perm)
        out, outf = torch.empty_like(k1_d), torch.empty_like(k1_d)
        q.apply_map_planned(plan, perm, k1_d, out, q.workspace())
        q.run_fused_planned(plan, gates, k1_d, outf, q.workspace())
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == ref.tobytes()
        assert outf.cpu().numpy().tobytes() == ref.tobytes()


def test_run_host_end_to_end(q):
    M = 16
    gates = wl.random_gates(64, M, 33)
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 33))
    ref = oracle.apply_map(oracle.build_map(gates, M), k1)
    for mode in (q.MATERIALISED, q.FUSED):
        k1_h = torch.from_numpy(k1.view(np.uint8).copy()).pin_memory()
        k2_h = torch.empty_like(k1_h).pin_memory()
        k1_d = torch.empty(k1_h.numel(), dtype=torch.uint8, device=DEV)
        k2_d = torch.empty_like(k1_d)
        perm = _new_perm(1 << M)
        q.run_host(gates, M, mode, k1_h, k2_h, k1_d, k2_d, perm, q.workspace(), dtype="c64")
        assert k2_h.numpy().tobytes() == ref.tobytes(), mode


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_run_host_batch_overlapped(q, dtype):
    """Serving form: several different states end to end with overlapped
    copies and double-buffered device state; every step's k2 equals the
    oracle's, in both modes, for odd and even step counts."""
    M = 17
    gates = wl.random_gates(64, M, 44)
    e = 8 if dtype == "c64" else 16
    states = [wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 50 + i)) for i in range(5)]
    refs = [oracle.apply_map(oracle.build_map(gates, M), k) for k in states]
    k1_h = [torch.from_numpy(k.view(np.uint8).copy()).pin_memory() for k in states]
    k1_d = [torch.empty((1 << M) * e, dtype=torch.uint8, device=DEV) for _ in range(2)]
    k2_d = [torch.empty_like(k1_d[0]) for _ in range(2)]
    perm = _new_perm(1 << M)
    for mode in (q.MATERIALISED, q.FUSED):
        for ns in (1, 2, 5):
            k2_h = [torch.empty_like(k1_h[0]).pin_memory() for _ in range(ns)]
            q.run_host_batch(gates, M, mode, k1_h[:ns], k2_h, k1_d, k2_d, perm, q.workspace(),
                             dtype=dtype)
            for i in range(ns):
                assert k2_h[i].numpy().tobytes() == refs[i].tobytes(), (mode, ns, i)


def test_special_values_survive(q):
    """-0.0, NaN payloads, denormals, inf: moved as bits (R15)."""
    M = 11
    N = 1 << M
    k1 = wl.tagged_state("c64", N)
    bits = k1.view(np.uint32).reshape(-1, 2)
    bits[:8, 0] = [0x80000000, 0x7fc00001, 0xffc12345, 0x00000001, 0x7f800000, 0xff800000,
                   0x7fbfffff, 0x80000001]
    gates = wl.random_gates(33, M, 21)
    ref = oracle.apply_map(oracle.build_map(gates, M), k1)
    k1_d = _to_dev(k1)
    k2 = torch.empty_like(k1_d)
    q.run_fused(gates, M, k1_d, k2, dtype="c64")
    torch.cuda.synchronize()
    assert k2.cpu().numpy().tobytes() == ref.tobytes()


def test_max_gates_and_capacity_buckets(q):
    M = 14
    for n in (63, 64, 65, 256, 257, 1024, 1025, q.MAX_GATES):
        gates = wl.random_gates(n, M, n)
        perm = _new_perm(1 << M)
        q.build_map(gates, M, perm)
        torch.cuda.synchronize()
        assert np.array_equal(_perm_np(perm), oracle.build_map(gates, M)), n


def test_determinism_and_streams(q):
    M = 18
    gates = wl.random_gates(64, M, 2)
    outs = []
    for i in range(3):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            p = _new_perm(1 << M)
            q.build_map(gates, M, p, stream=s)
        s.synchronize()
        outs.append(_perm_np(p).copy())
    assert all(np.array_equal(outs[0], o) for o in outs)


# -------------------------------------------------------- BASELINE configs
def test_cfg1_full(q):
    cfg = wl.CONFIGS["cfg1"]
    gates, k1 = cfg.gates(), wl.make_state(cfg.state)
    perm_ref = oracle.build_map(gates, cfg.M)
    assert perm_ref.tolist() == [0, 1, 7, 6, 4, 2, 3, 5]       # tests/golden/cfg1_perm.txt
    k1_d = _to_dev(k1)
    perm = _new_perm(8)
    q.build_map(gates, cfg.M, perm)
    k2, k2f = torch.empty_like(k1_d), torch.empty_like(k1_d)
    q.apply_map(perm, cfg.M, k1_d, k2, dtype="c64")
    q.run_fused(gates, cfg.M, k1_d, k2f, dtype="c64")
    torch.cuda.synchronize()
    ref = oracle.apply_map(perm_ref, k1)
    assert np.array_equal(_perm_np(perm), perm_ref)
    assert k2.cpu().numpy().tobytes() == ref.tobytes() == k2f.cpu().numpy().tobytes()


def test_cfg2_full(q):
    cfg = wl.CONFIGS["cfg2"]
    gates, k1 = cfg.gates(), wl.make_state(cfg.state)
    perm_ref = oracle.build_map(gates, cfg.M)
    ref = oracle.apply_map(perm_ref, k1)
    assert oracle.accumulate(gates, k1).tobytes() == ref.tobytes()
    k1_d = _to_dev(k1)
    perm = _new_perm(cfg.N)
    q.build_map(gates, cfg.M, perm)
    k2, k2f = torch.empty_like(k1_d), torch.empty_like(k1_d)
    q.apply_map(perm, cfg.M, k1_d, k2, dtype="c64")
    q.run_fused(gates, cfg.M, k1_d, k2f, dtype="c64")
    torch.cuda.synchronize()
    assert np.array_equal(_perm_np(perm), perm_ref)
    assert k2.cpu().numpy().tobytes() == ref.tobytes()
    assert k2f.cpu().numpy().tobytes() == ref.tobytes()


def _sample_indices(M, n=1 << 15, seed=0):
    N = 1 << M
    rng = np.random.default_rng(seed)
    edges = [0, 1, 31, 32, 1023, 1024, 1025, N // 2 - 1, N // 2, N - 1025, N - 1024, N - 2, N - 1]
    idx = np.concatenate([np.array(edges, dtype=np.uint64),
                          rng.integers(0, N, size=n, dtype=np.uint64)])
    return idx


# cfg3 / cfg4 / cfg5 at full size: every output against the oracle in
# tests/test_gpu_fullsize.py (these configs were sampled here before).


@pytest.mark.slow
def test_tagged_gather_m32(q):
    """Index-tagged k1 at M = 32 (re bits = j, im bits = ~j): k2's real bits
    must equal perm[i] for every output (a gather check at full size that
    needs no host copy of k1)."""
    M, N = 32, 1 << 32
    gates = wl.CONFIGS["cfg5"].gates()
    host = np.empty(1 << 28, dtype=np.complex64)
    k1_d = torch.empty(N * 8, dtype=torch.uint8, device=DEV)
    for s in range(0, N, 1 << 28):
        wl.fill_tagged("c64", host.ctypes.data, s, 1 << 28)
        k1_d[s * 8:(s + (1 << 28)) * 8].copy_(torch.from_numpy(host.view(np.uint8)))
    k2_d = torch.empty_like(k1_d)
    q.run_fused(gates, M, k1_d, k2_d, dtype="c64")
    perm_d = torch.empty(N, dtype=torch.int32, device=DEV)
    q.build_map(gates, M, perm_d)
    torch.cuda.synchronize()
    words = k2_d.view(torch.int32).view(-1, 2)
    for s in range(0, N, 1 << 28):
        w = words[s:s + (1 << 28)]
        assert torch.equal(w[:, 0], perm_d[s:s + (1 << 28)])
        assert torch.equal(w[:, 1], ~perm_d[s:s + (1 << 28)])
    idx = _sample_indices(M, 4096, 5)
    src = oracle.walk_many(gates, idx)
    it = torch.from_numpy(idx.astype(np.int64)).to(DEV)
    assert np.array_equal(words[:, 0].index_select(0, it).cpu().numpy().view(np.uint32)
                          .astype(np.uint64), src)
    torch.cuda.empty_cache()


@pytest.mark.parametrize("M", [16, 21])
def test_structured_circuits(q, M):
    """Circuits whose plans degenerate: gates only on high bits (whole blocks
    move, every sector's readers are one output run), only on low bits
    (in-run shuffles), the ripple cascade, NOT-only, and the empty list --
    every call (natural and planned, both dtypes) equals the oracle."""
    rng = np.random.default_rng(M)

    def rand_on(bits, n):
        rows = []
        for _ in range(n):
            kind = int(rng.integers(3))
            b = rng.choice(bits, size=1 + kind, replace=False)
            rows.append(wl.gate(kind, int(b[0]), *[int(x) for x in b[1:]]))
        return wl.gates_array(rows)

    circuits = {
        "high": rand_on(list(range(M - 6, M)), 40),
        "low": rand_on(list(range(0, 6)), 40),
        "ripple": wl.ripple_gates(M, 3 * (M - 2)),
        "not_only": wl.gates_array([wl.gate(wl.NOT, int(t)) for t in rng.integers(0, M, 9)]),
        "empty": wl.gates_array([]),
    }
    for name, gates in circuits.items():
        for dtype in ("c64", "c128"):
            k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 70 + M))
            perm_ref = oracle.build_map(gates, M)
            ref = oracle.apply_map(perm_ref, k1)
            k1_d = _to_dev(k1)
            perm = _new_perm(1 << M)
            q.build_map(gates, M, perm)
            torch.cuda.synchronize()
            assert np.array_equal(_perm_np(perm), perm_ref), name
            plan = q.plan_create(gates, M, dtype)
            for natural in (1, 0):
                plan.flags = natural
                outs = [torch.empty_like(k1_d) for _ in range(3)]
                pm = _new_perm(1 << M)
                q.apply_map_planned(plan, perm, k1_d, outs[0], q.workspace())
                q.run_fused_planned(plan, gates, k1_d, outs[1], q.workspace())
                q.map_gather_planned(plan, gates, pm, k1_d, outs[2], q.workspace())
                torch.cuda.synchronize()
                for o in outs:
                    assert o.cpu().numpy().tobytes() == ref.tobytes(), (name, dtype, natural)
                assert np.array_equal(_perm_np(pm), perm_ref), (name, dtype, natural)


@pytest.mark.parametrize("M,natural", [(16, 1), (16, 0), (20, 1), (18, 4)])   # 4: two-kernel step
def test_graphs_replay_planned_calls(q, M, natural):
    """CUDA graphs of repeated planned calls (launch-bound small states):
    replaying the recorded steps gives the oracle's bytes, for map + gather,
    fused and apply, natural and plan order, one- and two-kernel map + gather."""
    gates = wl.random_gates(64, M, 1700 + M)
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 4 + M))
    perm_ref = oracle.build_map(gates, M)
    ref = oracle.apply_map(perm_ref, k1)
    k1_d = _to_dev(k1)
    plan = q.plan_create(gates, M, "c64")
    plan.flags = natural
    ws = q.workspace()
    pm = _new_perm(1 << M)
    for call in (q.GRAPH_MAP_GATHER, q.GRAPH_FUSED, q.GRAPH_APPLY):
        out = torch.empty_like(k1_d)
        if call == q.GRAPH_APPLY:
            q.build_map(gates, M, pm)
        g = q.Graph(plan, gates, call, pm, k1_d, out, ws, reps=3)
        out.zero_()
        torch.cuda.synchronize()
        g.launch()
        g.launch()
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == ref.tobytes(), call
        if call == q.GRAPH_MAP_GATHER:
            assert np.array_equal(_perm_np(pm), perm_ref)
        g.close()
    if natural & q.PLAN_SPLIT:                            # no workspace: round-robin chunks
        out, pm2 = torch.empty_like(k1_d), _new_perm(1 << M)
        q.map_gather_planned(plan, gates, pm2, k1_d, out, None)
        assert q.last_launch_count() == 2
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == ref.tobytes()
        assert np.array_equal(_perm_np(pm2), perm_ref)


@pytest.mark.parametrize("dtype,M", [("c64", 13), ("c64", 17), ("c64", 22), ("c128", 12),
                                     ("c128", 19)])
def test_local_tiles_staged_in_shared_memory(q, M, dtype):
    """Circuits that keep locality (every target and SWAP bit below the tile,
    controls anywhere, phase steps included): the plan flags them and the
    TMA-staged shared-memory kernel runs -- same map and k2 bytes as the
    oracle; a circuit with one target above the tile does not take it."""
    T = 13 if dtype == "c64" else 12
    rng = np.random.default_rng(M + T)
    rows = []
    for _ in range(70):
        kind = int(rng.integers(7))
        nc = 1 if kind == 6 else kind % 3
        t = int(rng.integers(T))
        others = [b for b in range(M) if b != t] if kind != 6 else [b for b in range(T) if b != t]
        cs = rng.choice(others, size=nc, replace=False)
        rows.append(wl.gate(kind, t, *[int(c) for c in cs]))
    gates = wl.gates_array(rows)
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 30 + M))
    perm_ref, signs_ref = oracle.build_map_signed(gates, M)
    ref = oracle.apply_map_signed(perm_ref, signs_ref, k1)
    plain = np.ascontiguousarray(gates[(gates[:, 0] < 3) | (gates[:, 0] == 6)])
    perm_plain = oracle.build_map(plain, M)
    ref_plain = oracle.apply_map(perm_plain, k1)
    k1_d = _to_dev(k1)
    plan = q.plan_create(gates, M, dtype)
    assert plan.flags & 2
    out = torch.empty_like(k1_d)
    q.run_fused_planned(plan, gates, k1_d, out, q.workspace())
    assert q.last_kernel() == "qsim_jit_local"
    pm, out2 = _new_perm(1 << M), torch.empty_like(k1_d)
    q.map_gather_planned(q.plan_create(plain, M, dtype), plain, pm, k1_d, out2, q.workspace())
    assert q.last_kernel() == "qsim_jit_local"
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == ref.tobytes()
    assert out2.cpu().numpy().tobytes() == ref_plain.tobytes()
    assert np.array_equal(_perm_np(pm), perm_plain)
    # a target above the tile: the plan is not local and the generic kernels run
    if M == T:
        return
    far = np.concatenate([plain, wl.gates_array([wl.gate(wl.CNOT, M - 1, 0)])])
    plan_far = q.plan_create(far, M, dtype)
    assert not (plan_far.flags & 2)
    plan.flags |= 2                                   # a stale plan: re-checked on the gates
    out3 = torch.empty_like(k1_d)
    q.run_fused_planned(plan, far, k1_d, out3, q.workspace())
    assert q.last_kernel() != "qsim_jit_local"
    torch.cuda.synchronize()
    assert out3.cpu().numpy().tobytes() == oracle.apply_map(oracle.build_map(far, M), k1).tobytes()


# qsim_plan_tune / qsim_plan_tune_ex MEASURE / MEASURE for the planned apply
@pytest.mark.parametrize("effort", [None, 1, 0x101])
def test_plan_tune_keeps_a_valid_plan(q, effort):
    """qsim_plan_tune measures plan variants and keeps one: the result of its
    own runs and of the tuned plan afterwards equal the oracle's bytes."""
    M = 20
    gates = wl.random_gates(64, M, 8)
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 8))
    perm_ref = oracle.build_map(gates, M)
    ref = oracle.apply_map(perm_ref, k1)
    k1_d = _to_dev(k1)
    plan = q.plan_create(gates, M, "c64")
    plan.flags &= ~1
    pm, out = _new_perm(1 << M), torch.empty_like(k1_d)
    chosen = q.plan_tune(plan, gates, pm, k1_d, out, q.workspace(), effort=effort)
    assert 0 <= chosen % 8 <= 5 and chosen < 16
    assert bool(chosen & 8) == bool(plan.flags & q.PLAN_SPLIT)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == ref.tobytes()
    assert np.array_equal(_perm_np(pm), perm_ref)
    out2 = torch.empty_like(k1_d)
    q.run_fused_planned(plan, gates, k1_d, out2, q.workspace())
    torch.cuda.synchronize()
    assert out2.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.slow
def test_plan_tune_tail_order_stage(q):
    """Above the L2 (M = 25, 256 MB state) the tuner's third stage reorders the
    counter bits above the sector cover at run time: the kept plan is a
    valid order (a permutation fixing the kept low bits) and every output of
    map + gather, fused and apply with it equals the oracle."""
    import oracle.parallel as opar
    M = 25
    gates = wl.random_gates(64, M, 4)
    k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 25))
    perm_ref = opar.build_map(gates, M)
    ref = opar.apply_map(perm_ref, k1)
    k1_d = _to_dev(k1)
    plan = q.plan_create(gates, M, "c64")
    assert not (plan.flags & 1)
    pm, out = _new_perm(1 << M), torch.empty_like(k1_d)
    q.plan_tune(plan, gates, pm, k1_d, out, q.workspace())
    sig = list(plan.sigma)[:M]
    assert sorted(sig) == list(range(M)) and sig[:3] == [0, 1, 2]
    for run in ("mg", "fu", "ap"):
        out.fill_(0)
        if run == "mg":
            pm.fill_(-1)
            q.map_gather_planned(plan, gates, pm, k1_d, out, q.workspace())
        elif run == "fu":
            q.run_fused_planned(plan, gates, k1_d, out, q.workspace())
        else:
            q.apply_map_planned(plan, pm, k1_d, out, q.workspace())
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == ref.tobytes(), run
        assert np.array_equal(_perm_np(pm), perm_ref)


def test_plain_run_fused_concurrent_streams(q):
    """The plain qsim_run_fused keeps one chunk ticket per stream: two
    circuits run concurrently on two streams, repeatedly, give the oracle's
    bytes."""
    M = 18
    cases = []
    for sd in (1, 2):
        gates = wl.random_gates(60, M, 70 + sd)
        k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, sd))
        cases.append((gates, _to_dev(k1), oracle.apply_map(oracle.build_map(gates, M), k1)))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty_like(c[1]) for c in cases]
    for _ in range(3):
        for (gates, k1_d, _), o, st in zip(cases, outs, streams):
            q.run_fused(gates, M, k1_d, o, stream=st, dtype="c64")
        torch.cuda.synchronize()
        for (_, _, ref), o in zip(cases, outs):
            assert o.cpu().numpy().tobytes() == ref.tobytes()


def test_aot_fallback_launch_shapes(q):
    """Without NVRTC (QSIM_NO_JIT=1, a subprocess: the switch is read once per
    process) the planned calls run the ahead-of-time kernels; every launch
    shape (CTA threads x gathers in flight) gives the oracle's bytes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QSIM_NO_JIT="1")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "aot_fallback_check.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "aot fallback ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.slow
def test_build_max_gates_full_size(q):
    """Maximum sizes together: M = 32 (2^32 outputs, perm 16 GiB) and the
    largest gate list the parameter bank takes (QSIM_MAX_GATES), through the
    NVRTC build kernel; sampled outputs against the oracle's walk, and the
    map is a bijection on the samples' images (no two sampled outputs share
    a source)."""
    M, n = 32, q.MAX_GATES
    gates = wl.random_gates(n, M, 404)
    perm = torch.empty(1 << M, dtype=torch.int32, device=DEV)
    q.build_map(gates, M, perm)
    torch.cuda.synchronize()
    idx = _sample_indices(M, 20000, 9)
    got = perm.index_select(0, torch.from_numpy(idx.astype(np.int64)).to(DEV)).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, oracle.walk_many(gates, idx.astype(np.uint64)).astype(np.uint32))
    assert len(np.unique(got)) == len(np.unique(idx))
    del perm
    torch.cuda.empty_cache()
