"""C ABI: the library loads, exports every symbol include/qsim.h declares, and
rejects invalid arguments before touching the GPU (CPU only)."""
import ctypes
import os
import re

import numpy as np
import pytest

import workloads as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qsim.h")


@pytest.fixture(scope="module")
def q():
    import __graft_entry__
    __graft_entry__.build_native()
    import paper_quant_ph_0308158_b200 as q
    return q


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qsim_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for fn in ("qsim_build_map", "qsim_apply_map", "qsim_run_fused", "qsim_strerror"):
        assert fn in names


def test_library_exports_every_declared_symbol(q):
    lib = ctypes.CDLL(q.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.qsim_abi_version() == 7


def test_strerror_covers_every_status(q):
    for code in (q.OK, q.EINVAL, q.ERANGE, q.EBIT, q.ECAP, q.EALIAS, q.ECUDA):
        assert q.lib().qsim_strerror(code).decode() != "unknown qsim status"


def _rc(fn, *args):
    return fn(*args)


FAKE = 1 << 20          # a 16-byte aligned, never-dereferenced "device" address


def test_validation_errors_without_gpu(q):
    L = q.lib()
    ok = np.ascontiguousarray(wl.gates_array([wl.gate(wl.CNOT, 0, 1)]))
    gp = ok.ctypes.data
    # M out of range
    assert L.qsim_build_map(gp, 1, 0, FAKE, None) == q.ERANGE
    assert L.qsim_build_map(gp, 1, 33, FAKE, None) == q.ERANGE
    assert L.qsim_apply_map(FAKE, 0, q.C64, FAKE, FAKE * 4, None) == q.ERANGE
    assert L.qsim_run_fused(gp, 1, 40, q.C64, FAKE, FAKE * 4, None) == q.ERANGE
    # gate count
    assert L.qsim_build_map(gp, -1, 4, FAKE, None) == q.ECAP
    assert L.qsim_build_map(gp, q.MAX_GATES + 1, 4, FAKE, None) == q.ECAP
    assert L.qsim_build_map(None, 3, 4, FAKE, None) == q.EINVAL
    # null / misaligned pointers, bad dtype
    assert L.qsim_build_map(gp, 1, 4, None, None) == q.EINVAL
    assert L.qsim_build_map(gp, 1, 4, FAKE + 4, None) == q.EINVAL
    assert L.qsim_apply_map(None, 4, q.C64, FAKE, FAKE * 4, None) == q.EINVAL
    assert L.qsim_apply_map(FAKE, 4, 7, FAKE, FAKE * 4, None) == q.EINVAL
    assert L.qsim_run_fused(gp, 1, 4, q.C64, FAKE + 8, FAKE * 4, None) == q.EINVAL
    # range
    assert L.qsim_build_map_range(gp, 1, 4, 10, 7, FAKE, None) == q.ERANGE
    assert L.qsim_run_fused_range(gp, 1, 4, q.C64, 17, 0, FAKE, FAKE * 4, None) == q.ERANGE
    # bad walk selector
    assert L.qsim_build_map_ex(gp, 1, 4, 0, 16, FAKE, 9, None) == q.EINVAL
    # aliasing k1/k2 and perm/k2
    assert L.qsim_run_fused(gp, 1, 4, q.C64, FAKE, FAKE + 64, None) == q.EALIAS
    assert L.qsim_apply_map(FAKE, 4, q.C64, FAKE * 4, FAKE + 32, None) == q.EALIAS
    assert L.qsim_apply_map(FAKE, 4, q.C128, FAKE * 4, FAKE * 4 + 128, None) == q.EALIAS
    # run_host: bad mode, missing perm workspace
    assert L.qsim_run_host(gp, 1, 4, q.C64, 5, FAKE, FAKE, FAKE, FAKE * 4, FAKE * 8, None,
                           None) == q.EINVAL
    assert L.qsim_run_host(gp, 1, 4, q.C64, 0, FAKE, FAKE, FAKE, FAKE * 4, None, None,
                           None) == q.EINVAL
    assert L.qsim_run_host(gp, 1, 4, q.C64, 0, FAKE, FAKE, FAKE, FAKE * 4, FAKE * 8, FAKE + 8,
                           None) == q.EINVAL


@pytest.mark.parametrize("bad,code", [
    ([7, 0, 255, 255], "EINVAL"),      # unknown kind
    ([6, 1, 1, 255], "EBIT"),          # SWAP of a bit with itself
    ([6, 1, 5, 255], "EBIT"),          # SWAP partner >= M
    ([4, 0, 0, 255], "EBIT"),          # CZ control == target
    ([5, 0, 1, 1], "EBIT"),            # CCZ duplicate control
    ([0, 4, 255, 255], "EBIT"),        # target >= M
    ([1, 0, 0, 255], "EBIT"),          # control == target
    ([1, 0, 9, 255], "EBIT"),          # control >= M
    ([2, 0, 1, 1], "EBIT"),            # duplicate control
    ([2, 2, 1, 2], "EBIT"),            # target among controls
])
def test_gate_validation(q, bad, code):
    g = np.ascontiguousarray(np.array([[1, 0, 1, 255], bad], dtype=np.uint8))
    rc = q.lib().qsim_build_map(g.ctypes.data, 2, 4, FAKE, None)
    assert rc == getattr(q, code)
    rc = q.lib().qsim_run_fused(g.ctypes.data, 2, 4, q.C64, FAKE, FAKE * 4, None)
    assert rc == getattr(q, code)


def test_plan_create_and_validation(q):
    """Plans are host-only: create them and check the validator (no launch)."""
    g = wl.CONFIGS["cfg5"].gates()
    plan = q.plan_create(g, 32, "c64")
    sig = list(plan.sigma)[:32]
    assert sorted(sig) == list(range(32)) and sig[:3] == [0, 1, 2]
    assert 10 <= plan.tile_log2 <= 13 and plan.tile_contained > 0.5   # sector cover first
    assert plan.chunk_log2 == 15 and plan.fused_chunk_log2 == 15 and plan.blocks_per_sm == 1
    assert plan.flags == 0                       # cfg5: sigma order pays
    # deterministic
    assert list(q.plan_create(g, 32, "c64").sigma) == list(plan.sigma)
    # L2-resident and effectively random circuits keep natural order; the
    # ripple cascade's sector-mates are close: sigma (measured 1.4x / 2.3x
    # faster map+gather / fused on cfg4)
    for name, natural in (("cfg2", True), ("cfg3", True), ("cfg4", False)):
        cfg = wl.CONFIGS[name]
        assert bool(q.plan_create(cfg.gates(), cfg.M, cfg.dtype).flags & 1) == natural, name
    L = q.lib()
    import ctypes
    bad = q.Plan.from_buffer_copy(plan)
    bad.sigma[2], bad.sigma[7] = bad.sigma[7], bad.sigma[2]          # moves a kept bit
    assert L.qsim_apply_map_planned(ctypes.byref(bad), FAKE, FAKE * 4, FAKE * 64, None, None) == q.EINVAL
    bad = q.Plan.from_buffer_copy(plan)
    bad.sigma[9] = bad.sigma[10]                                      # not a permutation
    assert L.qsim_apply_map_planned(ctypes.byref(bad), FAKE, FAKE * 4, FAKE * 64, None, None) == q.EINVAL
    bad = q.Plan.from_buffer_copy(plan)
    bad.chunk_log2 = 9
    assert L.qsim_apply_map_planned(ctypes.byref(bad), FAKE, FAKE * 4, FAKE * 64, None, None) == q.EINVAL
    bad = q.Plan.from_buffer_copy(plan)
    bad.fused_chunk_log2 = 9
    assert L.qsim_run_fused_planned(ctypes.byref(bad), g.ctypes.data, 64, FAKE * 4, FAKE * 64,
                                    None, None) == q.EINVAL
    bad = q.Plan.from_buffer_copy(plan)
    bad.ilp = 12
    assert L.qsim_apply_map_planned(ctypes.byref(bad), FAKE, FAKE * 4, FAKE * 64, None, None) == q.EINVAL
    bad = q.Plan.from_buffer_copy(plan)
    bad.blocks_per_sm = 0
    assert L.qsim_run_fused_planned(ctypes.byref(bad), g.ctypes.data, 64, FAKE * 4, FAKE * 64,
                                    None, None) == q.EINVAL
    # gates must validate against the plan's M
    assert L.qsim_run_fused_planned(ctypes.byref(plan), g.ctypes.data, 64, FAKE * 4, FAKE * 64,
                                    FAKE + 8, None) in (q.EINVAL,)
    with pytest.raises(q.QsimError):
        q.plan_create(g, 30, "c64")                                    # bit 31 >= M


def test_unused_control_slots_are_ignored(q):
    """NOT / CNOT may carry garbage in unused control slots (header contract):
    validation must not reject them.  We only check the validator, so use a
    range of count 0 (nothing is launched)."""
    g = np.ascontiguousarray(np.array([[0, 1, 200, 17], [1, 2, 0, 99]], dtype=np.uint8))
    assert q.lib().qsim_build_map_range(g.ctypes.data, 2, 3, 0, 0, FAKE, None) == q.OK


def test_jit_source_compiles_without_gpu(q):
    """The circuit-specialised build kernel is generated and NVRTC-compiled
    for sm_100a on the host (load/launch needs the GPU)."""
    L = q.lib()
    L.qsim_jit_check_compile.restype = ctypes.c_int
    for gates, M in ((wl.CONFIGS["cfg5"].gates(), 32), (wl.CONFIGS["cfg4"].gates(), 30),
                     (np.zeros((0, 4), np.uint8), 5), (wl.CONFIGS["cfg1"].gates(), 3)):
        g = np.ascontiguousarray(gates)
        rc = L.qsim_jit_check_compile(g.ctypes.data if len(g) else None, len(g), M)
        if rc != q.OK and "libnvrtc" in L.qsim_last_error().decode():
            pytest.skip("NVRTC not available here")
        assert rc == q.OK, L.qsim_last_error().decode()


def test_jit_build_thread_bits_source_compiles_without_gpu(q):
    """The build kernel's in-thread affine fast path."""
    L = q.lib()
    for gates, M in ((wl.CONFIGS["cfg5"].gates(), 32), (wl.random_gates(96, 14, 5), 22)):
        g = np.ascontiguousarray(gates)
        rc = L.qsim_jit_check_compile(g.ctypes.data, len(g), M)
        if rc != q.OK and "libnvrtc" in L.qsim_last_error().decode():
            pytest.skip("NVRTC not available here")
        assert rc == q.OK, L.qsim_last_error().decode()


def test_jit_fused_source_compiles_without_gpu(q):
    L = q.lib()
    for name in ("cfg5", "cfg3"):
        cfg = wl.CONFIGS[name]
        g = np.ascontiguousarray(cfg.gates())
        plan = q.plan_create(g, cfg.M, cfg.dtype)
        rc = L.qsim_jit_check_compile_planned(ctypes.byref(plan), g.ctypes.data, len(g))
        if rc != q.OK and "libnvrtc" in L.qsim_last_error().decode():
            pytest.skip("NVRTC not available here")
        assert rc == q.OK, L.qsim_last_error().decode()


def test_jit_kron_source_compiles_without_gpu(q):
    L = q.lib()
    # cfg5: the in-thread layout (hoisted product) is generated; M = 40 / 63:
    # 64 bit planes; phases: the sign plane in both paths
    for gates, M, dt in ((wl.CONFIGS["cfg5"].gates(), 32, q.C64), (wl.CONFIGS["cfg4"].gates(), 30, q.C128),
                         (wl.random_gates(10, 9, 1), 9, q.C64), (wl.random_gates(64, 40, 80), 40, q.C64),
                         (wl.random_gates_ext(48, 63, 2), 63, q.C128),
                         (wl.random_gates_ext(64, 24, 8), 24, q.C64)):
        g = np.ascontiguousarray(gates)
        rc = L.qsim_jit_check_compile_kron(g.ctypes.data, len(g), M, dt)
        if rc != q.OK and "libnvrtc" in L.qsim_last_error().decode():
            pytest.skip("NVRTC not available here")
        assert rc == q.OK, L.qsim_last_error().decode()


def test_kron_validation(q):
    L = q.lib()
    g = np.ascontiguousarray(wl.random_gates(5, 8, 1))
    qd = np.zeros(4 * 8)
    assert L.qsim_run_fused_kron(g.ctypes.data, 5, 8, q.C64, None, 0, 256, FAKE, 0, None) == q.EINVAL
    assert L.qsim_run_fused_kron(g.ctypes.data, 5, 8, q.C64, qd.ctypes.data, 0, 257, FAKE, 0,
                                 None) == q.ERANGE
    assert L.qsim_run_fused_kron(g.ctypes.data, 5, 8, 9, qd.ctypes.data, 0, 256, FAKE, 0,
                                 None) == q.EINVAL
    assert L.qsim_run_fused_kron(g.ctypes.data, 5, 8, q.C64, qd.ctypes.data, 0, 256, FAKE, 4,
                                 None) == q.EINVAL      # no such walk
    assert L.qsim_run_fused_kron(g.ctypes.data, 5, 8, q.C64, qd.ctypes.data, 0, 0, FAKE, 0,
                                 None) == q.OK
    # M > 32 only here (input on the fly, 64-bit addresses): up to 63
    g40 = np.ascontiguousarray(wl.random_gates(5, 40, 1))
    q40 = np.zeros(4 * 64)
    for M, want in ((40, q.OK), (63, q.OK), (64, q.ERANGE), (0, q.ERANGE)):
        gg = g40 if M >= 40 else g
        assert L.qsim_run_fused_kron(gg.ctypes.data, 5, M, q.C64, q40.ctypes.data, 1 << 35, 0,
                                     FAKE, 0, None) == (want if M != 0 else q.ERANGE), M
    assert L.qsim_run_fused_kron(g40.ctypes.data, 5, 40, q.C64, q40.ctypes.data, (1 << 40) - 3, 4,
                                 FAKE, 0, None) == q.ERANGE
    assert L.qsim_build_map(g40.ctypes.data, 5, 40, FAKE, None) == q.ERANGE   # maps stay M <= 32


def test_sector_cover_plan_matches_an_independent_sample(q):
    """Host logic of the plan's sector cover (qsim_plan_create): sigma is a
    permutation keeping the output-run bits in place, its first tile_log2
    counter bits are the cover, and the library's sampled containment agrees
    with a fresh sample computed from the oracle's walk (readers of the
    sector-mates of s = perm(i): g(s ^ r), g = walk of the reversed gate list,
    the inverse map)."""
    import oracle
    for name, dtype in (("cfg5", "c64"), ("cfg4", "c64"), ("cfg3", "c128")):
        cfg = wl.CONFIGS[name]
        g = cfg.gates()
        plan = q.plan_create(g, cfg.M, dtype)
        e = 8 if dtype == "c64" else 16
        T = plan.tile_log2
        assert 10 <= T <= 13
        sig = list(plan.sigma)[:cfg.M]
        assert sorted(sig) == list(range(cfg.M))
        keep = 3 if e == 8 else 2
        assert sig[:keep] == list(range(keep))
        assert sig[:T] == sorted(sig[:T])            # the cover, ascending
        V = 0
        for b in sig[:T]:
            V |= 1 << b
        rng = np.random.default_rng(123)
        i = rng.integers(0, 1 << cfg.M, size=3000, dtype=np.uint64)
        s = oracle.walk_many(g, i)
        rev = np.ascontiguousarray(g[::-1])
        hits = tot = 0
        for r in range(1, 32 // e):
            d = oracle.walk_many(rev, s ^ np.uint64(r)) ^ i
            hits += int(np.count_nonzero((d & ~np.uint64(V)) == 0))
            tot += d.size
        assert abs(hits / tot - plan.tile_contained) < 0.05, (name, hits / tot, plan.tile_contained)


def test_phase_gates_rejected_where_only_a_map_is_produced(q):
    """A circuit with Z / CZ / CCZ has rows of value -1: the calls whose only
    output is a uint32 map refuse it (EINVAL) before any launch; SWAP passes
    validation; the signed build checks its alignment rule."""
    L = q.lib()
    ph = np.ascontiguousarray(np.array([[1, 0, 1, 255], [4, 2, 0, 255]], dtype=np.uint8))
    sw = np.ascontiguousarray(np.array([[6, 0, 3, 255]], dtype=np.uint8))
    assert L.qsim_build_map(ph.ctypes.data, 2, 4, FAKE, None) == q.EINVAL
    assert L.qsim_build_map_ex(ph.ctypes.data, 2, 4, 0, 16, FAKE, q.WALK_JIT, None) == q.EINVAL
    plan = q.plan_create(ph, 4, "c64")                  # plans accept any valid circuit
    assert L.qsim_map_gather_planned(ctypes.byref(plan), ph.ctypes.data, 2, FAKE, FAKE * 4,
                                     FAKE * 64, None, None) == q.EINVAL
    assert L.qsim_run_host(ph.ctypes.data, 2, 4, q.C64, 0, FAKE, FAKE, FAKE, FAKE * 4, FAKE * 8,
                           None, None) == q.EINVAL
    assert L.qsim_build_map_signed(ph.ctypes.data, 2, 6, 16, 16, FAKE, FAKE * 4, None) == q.EINVAL
    assert L.qsim_build_map_signed(ph.ctypes.data, 2, 6, 0, 16, FAKE, None, None) == q.EINVAL
    assert L.qsim_build_map_signed(ph.ctypes.data, 2, 4, 0, 17, FAKE, FAKE * 4, None) == q.ERANGE
    assert L.qsim_apply_map_signed(FAKE, None, 16, 4, q.C64, FAKE * 4, FAKE * 8, None) == q.EINVAL
    # SWAP is a plain permutation: it validates (the EALIAS proves validation passed)
    rc = L.qsim_run_fused(sw.ctypes.data, 1, 4, q.C64, FAKE, FAKE, None)
    assert rc == q.EALIAS


def test_jit_sources_with_phase_and_swap_compile_without_gpu(q):
    """NVRTC accepts the generated kernels for the extended gate set (swap =
    variable renaming, phase = sign register) -- fused (planned) and kron."""
    L = q.lib()
    g = np.ascontiguousarray(wl.random_gates_ext(64, 20, 3))
    plan = q.plan_create(g, 20, "c64")
    rc = L.qsim_jit_check_compile_planned(ctypes.byref(plan), g.ctypes.data, len(g))
    if rc != q.OK and "libnvrtc" in L.qsim_last_error().decode():
        pytest.skip("NVRTC not available here")
    assert rc == q.OK, L.qsim_last_error().decode()
    for dt in (q.C64, q.C128):
        assert L.qsim_jit_check_compile_kron(g.ctypes.data, len(g), 20, dt) == q.OK, \
            L.qsim_last_error().decode()


def test_run_host_batch_validation(q):
    """The overlapped end-to-end call validates everything before any copy."""
    L = q.lib()
    g = np.ascontiguousarray(wl.random_gates(5, 10, 1))
    hosts = (ctypes.c_void_p * 2)(FAKE, FAKE)
    n = 1 << 10
    args = [g.ctypes.data, 5, 10, q.C64, 0, 2, ctypes.cast(hosts, ctypes.c_void_p),
            ctypes.cast(hosts, ctypes.c_void_p)]
    devs = [FAKE * 8, FAKE * 8 + n * 8, FAKE * 8 + 2 * n * 8, FAKE * 8 + 3 * n * 8]
    perm = FAKE * 8 + 4 * n * 8
    assert L.qsim_run_host_batch(*args, *devs, None, None) == q.EINVAL          # mode 0 needs perm
    assert L.qsim_run_host_batch(*args[:4], 2, 2, *args[6:], *devs, perm, None) == q.EINVAL
    bad = list(devs)
    bad[1] = devs[0] + 16                                                       # k1 buffers overlap
    assert L.qsim_run_host_batch(*args, *bad, perm, None) == q.EALIAS
    assert L.qsim_run_host_batch(*args[:5], 0, *args[6:], *devs, perm, None) == q.OK   # no steps
    nulls = (ctypes.c_void_p * 2)(FAKE, None)
    assert L.qsim_run_host_batch(*args[:6], ctypes.cast(nulls, ctypes.c_void_p), args[7], *devs,
                                 perm, None) == q.EINVAL


def test_graph_validation(q):
    L = q.lib()
    g = np.ascontiguousarray(wl.random_gates(5, 12, 1))
    plan = q.plan_create(g, 12, "c64")
    h = ctypes.c_void_p()
    assert L.qsim_graph_create(ctypes.byref(plan), g.ctypes.data, 5, 0, FAKE, FAKE * 4, FAKE * 8,
                               None, 0, ctypes.byref(h)) == q.EINVAL          # reps < 1
    assert L.qsim_graph_create(ctypes.byref(plan), g.ctypes.data, 5, 3, FAKE, FAKE * 4, FAKE * 8,
                               None, 1, ctypes.byref(h)) == q.EINVAL          # no such call
    assert L.qsim_graph_create(ctypes.byref(plan), g.ctypes.data, 5, 0, FAKE, FAKE * 4, FAKE * 8,
                               None, 1, None) == q.EINVAL
    assert L.qsim_graph_launch(None, None) == q.EINVAL
    assert L.qsim_graph_destroy(None) == q.OK


def test_plan_tune_validation(q):
    L = q.lib()
    g = np.ascontiguousarray(wl.random_gates(20, 16, 1))
    plan = q.plan_create(g, 16, "c64")
    chosen = ctypes.c_int32(-1)
    assert L.qsim_plan_tune(ctypes.byref(plan), g.ctypes.data, 20, FAKE, FAKE * 4, FAKE * 8, None,
                            None, ctypes.byref(chosen)) == q.EINVAL          # needs a workspace
    ph = np.ascontiguousarray(np.array([[4, 2, 0, 255]], dtype=np.uint8))
    plan2 = q.plan_create(ph, 16, "c64")
    assert L.qsim_plan_tune(ctypes.byref(plan2), ph.ctypes.data, 1, FAKE, FAKE * 4, FAKE * 8,
                            FAKE * 16, None, None) == q.EINVAL                # phase circuit
    for effort in (0, 3, -1, q.TUNE_APPLY, q.TUNE_APPLY | 3, 0x200 | q.TUNE_MEASURE):  # no such effort
        assert L.qsim_plan_tune_ex(ctypes.byref(plan), g.ctypes.data, 20, FAKE, FAKE * 4, FAKE * 8,
                                   FAKE * 16, None, effort, ctypes.byref(chosen)) == q.EINVAL
    assert L.qsim_plan_tune_ex(ctypes.byref(plan), g.ctypes.data, 20, FAKE, FAKE * 4, FAKE * 8,
                               None, None, q.TUNE_MEASURE, None) == q.EINVAL  # needs a workspace


def test_binding_checks_before_the_c_call(q):
    """The ctypes binding checks what the C ABI cannot see: device
    buffers must be CUDA tensors of at least the bytes the call writes, and
    the on-the-fly input's dtype follows its output tensor."""
    import torch
    g = wl.random_gates(5, 10, 1)
    with pytest.raises(ValueError, match="CUDA"):
        q.build_map(g, 10, torch.empty(1 << 10, dtype=torch.int32))          # host tensor
    with pytest.raises(ValueError, match="CUDA"):
        q.run_fused(g, 10, torch.empty(1 << 10, dtype=torch.complex64),
                    torch.empty(1 << 10, dtype=torch.complex64))
    qb = wl.random_qubits(10, 1, "c64")
    with pytest.raises(ValueError, match="dtype"):
        q.run_fused_kron(g, 10, qb, torch.empty(1 << 10, dtype=torch.complex128), dtype="c64")


def test_binding_wrappers_reach_their_checks(q):
    """Every wrapper that takes device buffers rejects host tensors with a
    ValueError before the C call (catches wrapper bugs without a GPU)."""
    import torch
    M = 12
    g = wl.random_gates(5, M, 2)
    plan = q.plan_create(g, M, "c64")
    k = torch.empty(1 << M, dtype=torch.complex64)
    p = torch.empty(1 << M, dtype=torch.int32)
    ws = torch.empty(q.WORKSPACE_BYTES, dtype=torch.uint8)
    calls = [lambda: q.apply_map(p, M, k, k), lambda: q.apply_map_planned(plan, p, k, k, ws),
             lambda: q.run_fused_planned(plan, g, k, k, ws),
             lambda: q.map_gather_planned(plan, g, p, k, k, ws),
             lambda: q.build_map_range(g, M, 0, 1 << M, p)]
    for c in calls:
        with pytest.raises(ValueError):
            c()


def test_header_constants_match_the_binding(q):
    """The plan flag and tuner-effort values the binding uses are the header's."""
    h = open(os.path.join(ROOT, "include", "qsim.h")).read()
    assert int(re.search(r"#define QSIM_PLAN_SPLIT (\d+)u", h).group(1)) == q.PLAN_SPLIT
    assert int(re.search(r"#define QSIM_WORKSPACE_BYTES (\d+)", h).group(1)) == q.WORKSPACE_BYTES
    assert int(re.search(r"QSIM_TUNE_MEASURE = (\d+)", h).group(1)) == q.TUNE_MEASURE
    assert int(re.search(r"QSIM_TUNE_PATIENT = (\d+)", h).group(1)) == q.TUNE_PATIENT
    assert int(re.search(r"QSIM_TUNE_APPLY = (0x[0-9a-f]+)", h).group(1), 16) == q.TUNE_APPLY
