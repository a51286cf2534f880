"""Full-size, element-by-element parity for BASELINE.json cfg3, cfg4 and cfg5.

Every one of the 2^26 / 2^30 / 2^32 outputs of every mode is compared with the
CPU oracle (perm as uint32, k2 as raw entry bytes; readings R14/R15):

* the oracle (oracle/qsim_oracle.c, single-threaded C, driven on disjoint
  output ranges from host threads by oracle/parallel.py) computes
  perm[i] = f_1(...f_n(i)) and k2[i] = k1[perm[i]] for all i (P:L35, P:L43,
  readings R1/R2) -- about 1.5 minutes per config on 16 host cores;
* the CUDA path runs through the C ABI: the plain calls of the north star
  (qsim_build_map, qsim_apply_map, qsim_run_fused), the planned calls with the
  default plan (qsim_plan_create) AND with the plan qsim_plan_tune keeps (the
  kernel instance bench.py times), and the end-to-end host-buffer call
  (qsim_run_host);
* the oracle's perm and k2 are copied to the device once and each mode's
  output is compared with them byte for byte (torch.equal on 512 MiB
  chunks); a failure names the mode and the first mismatching output index.
"""
import numpy as np
import pytest

import oracle
import oracle.parallel as opar
import workloads as wl

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DEV = "cuda:0"
CHUNK_BYTES = 1 << 29


@pytest.fixture(scope="module")
def q():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_native()
    import paper_quant_ph_0308158_b200 as q
    return q


def _compare(dev_u8, ref_u8, unit: int, label: str) -> None:
    """dev_u8 (the CUDA path's output) and ref_u8 (the oracle's, copied to the
    device once) are uint8 tensors; unit: bytes per entry."""
    assert dev_u8.numel() >= ref_u8.numel(), label
    for s in range(0, ref_u8.numel(), CHUNK_BYTES):
        e = min(ref_u8.numel(), s + CHUNK_BYTES)
        a, b = dev_u8[s:e], ref_u8[s:e]
        if not torch.equal(a, b):
            bad = (a.view(-1, unit) != b.view(-1, unit)).any(dim=1).nonzero()[0, 0].item()
            i = s // unit + bad
            pytest.fail(f"{label}: first mismatch at output {i} "
                        f"(got {dev_u8[i * unit:(i + 1) * unit].cpu().numpy().tobytes().hex()}, "
                        f"want {ref_u8[i * unit:(i + 1) * unit].cpu().numpy().tobytes().hex()})")


def _to_device(a: np.ndarray):
    out = torch.empty(a.nbytes, dtype=torch.uint8, device=DEV)
    flat = a.view(np.uint8).reshape(-1)
    for s in range(0, flat.size, 1 << 30):
        out[s:s + (1 << 30)].copy_(torch.from_numpy(flat[s:s + (1 << 30)]))
    return out


def _host_compare(got: np.ndarray, ref: np.ndarray, unit: int, label: str) -> None:
    a, b = got.view(np.uint8).reshape(-1), ref.view(np.uint8).reshape(-1)
    for s in range(0, b.size, CHUNK_BYTES):
        e = min(b.size, s + CHUNK_BYTES)
        if not np.array_equal(a[s:e], b[s:e]):
            bad = np.flatnonzero((a[s:e].reshape(-1, unit) != b[s:e].reshape(-1, unit)).any(axis=1))
            pytest.fail(f"{label}: first mismatch at output {s // unit + int(bad[0])}")


def _run_config(q, name):
    cfg = wl.CONFIGS[name]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    e = 8 if cfg.dtype == "c64" else 16
    # ---- the oracle over every output (host)
    k1_host = np.empty(N, dtype=wl.NP_DTYPE[cfg.dtype])
    wl.fill_state(cfg.state, k1_host.ctypes.data)
    perm_ref = opar.build_map(gates, M)
    k2_ref = opar.apply_map(perm_ref, k1_host)
    # the oracle's own sampled walk agrees with its materialised map (sanity)
    idx = np.array([0, 1, N // 2, N - 1], dtype=np.uint64)
    assert np.array_equal(oracle.walk_many(gates, idx), perm_ref[idx.astype(np.int64)])

    # ---- device buffers (the oracle's perm and k2 are copied to the device
    # once, so each mode is compared there, byte for byte)
    k1 = _to_device(k1_host)
    perm_ref_d = _to_device(perm_ref)
    k2_ref_d = _to_device(k2_ref)
    k2 = torch.empty(N * e, dtype=torch.uint8, device=DEV)
    perm = torch.empty(N, dtype=torch.int32, device=DEV)
    ws = q.workspace()
    perm_u8 = perm.view(torch.uint8)

    def check_perm(label):
        torch.cuda.synchronize()
        _compare(perm_u8, perm_ref_d, 4, f"{name} {label} perm")

    def check_k2(label):
        torch.cuda.synchronize()
        _compare(k2, k2_ref_d, e, f"{name} {label} k2")
        k2.fill_(0xA5)                                  # stale bytes cannot pass the next mode

    # the north star's plain calls
    perm.fill_(-1)
    q.build_map(gates, M, perm)
    check_perm("qsim_build_map")
    q.apply_map(perm, M, k1, k2, dtype=cfg.dtype)
    check_k2("qsim_apply_map")
    q.run_fused(gates, M, k1, k2, dtype=cfg.dtype)
    check_k2("qsim_run_fused")
    # the planned calls with the default plan
    plan = q.plan_create(gates, M, cfg.dtype)
    q.apply_map_planned(plan, perm, k1, k2, ws)
    check_k2(f"qsim_apply_map_planned (plan_create, sigma {list(plan.sigma)[:8]}...)")
    q.run_fused_planned(plan, gates, k1, k2, ws)
    check_k2("qsim_run_fused_planned (plan_create)")
    perm.fill_(-1)
    q.map_gather_planned(plan, gates, perm, k1, k2, ws)
    check_perm("qsim_map_gather_planned (plan_create)")
    check_k2("qsim_map_gather_planned (plan_create)")
    # the plan bench.py times (qsim_plan_tune keeps the fastest variant)
    tuned = q.plan_create(gates, M, cfg.dtype)
    variant = q.plan_tune(tuned, gates, perm, k1, k2, ws)
    label = f"tuned plan (variant {variant}, sigma {list(tuned.sigma)[:13]}, chunk {tuned.fused_chunk_log2})"
    perm.fill_(-1)
    k2.fill_(0xA5)
    q.map_gather_planned(tuned, gates, perm, k1, k2, ws)
    check_perm("qsim_map_gather_planned " + label)
    check_k2("qsim_map_gather_planned " + label)
    if not (tuned.flags & 1):
        # the tuned order in the other map + gather mode (one kernel storing perm
        # in plan order <-> gather then natural-order build, QSIM_PLAN_SPLIT)
        other = q.Plan.from_buffer_copy(tuned)
        other.flags ^= q.PLAN_SPLIT
        perm.fill_(-1)
        q.map_gather_planned(other, gates, perm, k1, k2, ws)
        check_perm(f"qsim_map_gather_planned (flags {other.flags}) " + label)
        check_k2(f"qsim_map_gather_planned (flags {other.flags}) " + label)
    q.run_fused_planned(tuned, gates, k1, k2, ws)
    check_k2("qsim_run_fused_planned " + label)
    q.apply_map_planned(tuned, perm, k1, k2, ws)
    check_k2("qsim_apply_map_planned " + label)
    # the plan bench.py's two-call mode times (tuned for the planned apply)
    ap = q.plan_create(gates, M, cfg.dtype)
    if not (ap.flags & 1):
        perm.fill_(-1)
        q.plan_tune(ap, gates, perm, k1, k2, ws, effort=q.TUNE_MEASURE | q.TUNE_APPLY)
        check_perm("qsim_plan_tune_ex(APPLY) map")
        k2.fill_(0xA5)
        q.apply_map_planned(ap, perm, k1, k2, ws)
        check_k2(f"qsim_apply_map_planned (apply-tuned plan, sigma {list(ap.sigma)[:13]})")
    # end to end from host buffers (the e2e leg of bench.py)
    k2_host = np.empty_like(k1_host)
    for mode in (q.MATERIALISED, q.FUSED):
        k2_host.view(np.uint8)[:] = 0xA5
        q.run_host(gates, M, mode, k1_host, k2_host, k1, k2, perm, ws, dtype=cfg.dtype)
        _host_compare(k2_host, k2_ref, e, f"{name} qsim_run_host mode {mode} k2 (host)")
    del k2_host, perm_ref_d, k2_ref_d
    return cfg, perm, k1, k2


def test_cfg3_every_output(q):
    """cfg3: M = 26, 256 random gates, complex128 (materialised map then gather)."""
    _run_config(q, "cfg3")
    torch.cuda.empty_cache()


def test_cfg4_every_output(q):
    """cfg4: M = 30, 256-gate ripple cascade, complex64 (fused vs materialised)."""
    _run_config(q, "cfg4")
    torch.cuda.empty_cache()


def test_cfg5_every_output(q):
    """cfg5: M = 32, 64 random gates, complex64 -- the bench's workload."""
    cfg, perm, k1, k2 = _run_config(q, "cfg5")
    # group identity at full size as well: perm(rev G)[perm(G)[i]] == i
    del k1, k2
    torch.cuda.empty_cache()
    q.build_map(cfg.gates(), cfg.M, perm)
    rev = torch.empty_like(perm)
    q.build_map(cfg.gates()[::-1].copy(), cfg.M, rev)
    step = 1 << 28
    for s in range(0, cfg.N, step):
        p = perm[s:s + step].to(torch.int64) & 0xFFFFFFFF
        comp = rev.index_select(0, p).to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(comp, torch.arange(s, s + step, device=DEV, dtype=torch.int64))
    torch.cuda.empty_cache()
