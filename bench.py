#!/usr/bin/env python
"""bench.py -- throughput of the Burger permutation-map hot path on B200.

Metric (BASELINE.json): "state entries/sec and achieved HBM GB/s (fraction of
8 TB/s) for map+gather at M=32".  Workload: config 5 (M = 32, 64 random
NOT/CNOT/CCNOT gates, seed 4, complex64 Gaussian normalised state).

One step = the whole hot path over the 2^32-entry state, materialised:
qsim_map_gather_planned computes the composite map perm (uint32, stored:
"save information about the unitary matrix") and the state transform
k2[i] = k1[perm[i]] with kernels compiled for the circuit -- one
kernel storing perm in plan order, or (plan flag QSIM_PLAN_SPLIT, what
qsim_plan_tune keeps on cfg5) the planned gather then the natural-order
build; the plan is measured once, outside the timed region.  The
two-call form (qsim_build_map then qsim_apply_map_planned) and the fused
mode (qsim_run_fused_planned: the map recomputed, no perm) are timed in
their own loops and reported under "modes".  Inputs are larger than L2
(80 GiB working set vs 126 MB L2), so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5]
    python bench.py --impl reference      # the oracle, timed on host cores

With torchrun (N > 1) every rank runs its own replica of the workload on its
own GPU (no data-path collective; "scaling": "weak"); timing is the max over
ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "state entries/sec and achieved HBM GB/s (fraction of 8 TB/s) for map+gather at M=32"
FALLBACK_HBM_GBS = 6650.0       # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="qsim", choices=["qsim", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--cpu-sample-log2", type=int, default=29,
                    help="outputs in the oracle's bounded sample (log2)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config: str, kernel: str):
    """dram read+write bytes per launch from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self._stop = [], 0, threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        rs = [n for b, n in self.REASONS.items() if self.reasons & b and b != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": rs, "samples": len(self.samples)}


def dist_setup():
    """(world, rank, local_rank) from the torchrun environment (no package
    import: the reference arm must not load libqsim.so)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ------------------------------------------------------------ cpu baseline
def cpu_oracle_rate(gates, k1_host: np.ndarray, start: int, count: int, threads: int):
    """The oracle as it stands (build then apply, single-threaded C) over the
    output portion [start, start+count), split across `threads` host threads
    on disjoint sub-ranges (ctypes releases the GIL).  Returns (entries/s, s)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    per = (count + threads - 1) // threads
    out = np.empty(count, dtype=k1_host.dtype)

    def work(t):
        a = start + t * per
        b = min(start + count, a + per)
        if a >= b:
            return
        perm = oracle.build_map(gates, k1_host.shape[0].bit_length() - 1, a, b - a)
        out[a - start:b - start] = oracle.apply_map(perm, k1_host)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    dt = time.perf_counter() - t0
    return count / dt, dt


def verify_sample(gates, M, e, perm, k2, k1_host, cfg, dev, n=1 << 16, seed=2025):
    """Post-timing check of the timed step: 2^16 seeded output indices (plus
    the first and last 64) of perm and k2 against the oracle's walk
    (oracle.walk_many) and k1 at the oracle's sources (the host copy, or the
    counter-based generator entry by entry when no host copy exists)."""
    import torch
    import oracle
    import workloads as wl
    N = 1 << M
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([np.arange(min(64, N)), np.arange(max(0, N - 64), N),
                                    rng.integers(0, N, size=n)]).astype(np.uint64))
    src = oracle.walk_many(gates, idx)
    it = torch.from_numpy(idx.astype(np.int64)).to(dev)
    got_perm = perm.index_select(0, it).cpu().numpy().view(np.uint32).astype(np.uint64)
    got_k2 = k2.view(-1, e).index_select(0, it).cpu().numpy()
    if k1_host is not None:
        want = k1_host.numpy().reshape(-1, e)[src.astype(np.int64)]
    else:
        scale = cfg.state.scale()
        want = np.stack([wl.make_state(cfg.state, int(j), 1, scale=scale).view(np.uint8)
                         for j in src])
    ok_perm = bool(np.array_equal(got_perm, src))
    ok_k2 = bool(np.array_equal(got_k2, want))
    return {"ok": ok_perm and ok_k2, "outputs_checked": int(idx.size), "perm_equal": ok_perm,
            "k2_bytes_equal": ok_k2,
            "how": "after the timed loop: perm[i] and k2[i] at 2^16 seeded outputs (+ first/last 64) "
                   "vs oracle.walk_many (single-threaded C walk, P:L43) and k1[perm_oracle[i]]"}


def host_info():
    info = {"cpu_model": None, "host_ram_gb": None, "nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["cpu_model"] = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    info["host_ram_gb"] = round(int(ln.split()[1]) / (1 << 20), 1)
                    break
    except OSError:
        pass
    return info


def cpu_single_core(gates, k1_np: np.ndarray, count: int):
    """The oracle (build walk + apply gather) on ONE host core (the process
    pinned to core 0 for the call, like taskset -c 0), outputs [0, count)."""
    import oracle
    old = os.sched_getaffinity(0)
    core = min(old)
    os.sched_setaffinity(0, {core})
    try:
        t0 = time.perf_counter()
        perm = oracle.build_map(gates, k1_np.shape[0].bit_length() - 1, 0, count)
        oracle.apply_map(perm, k1_np)
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, old)
    return count / dt, dt, core


def cpu_accumulate(gates, k1_np: np.ndarray, n_gates: int):
    """The paper's "basic accumulation method" (oracle_accumulate,
    gate-by-gate pair swaps over the whole state) on one core, for the first
    n_gates steps over the full state, in place; the same steps then run in
    reverse order (each step is an involution), which restores k1
    exactly (checked on a sample).  Returns entry-steps/s and seconds."""
    import ctypes
    import oracle
    lib = oracle._load()
    M = k1_np.shape[0].bit_length() - 1
    e = k1_np.dtype.itemsize
    g = np.ascontiguousarray(gates[:n_gates], dtype=np.uint8)
    gr = np.ascontiguousarray(g[::-1])
    probe = np.array(k1_np[:: max(1, k1_np.shape[0] // 4096)], copy=True)
    old = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {min(old)})
    try:
        t0 = time.perf_counter()
        lib.oracle_accumulate(g.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), n_gates, M, e,
                              k1_np.ctypes.data)
        dt = time.perf_counter() - t0
        lib.oracle_accumulate(gr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), n_gates, M, e,
                              k1_np.ctypes.data)
    finally:
        os.sched_setaffinity(0, old)
    after = np.array(k1_np[:: max(1, k1_np.shape[0] // 4096)], copy=True)
    restored = bool(np.array_equal(probe.view(np.uint8), after.view(np.uint8)))
    return k1_np.shape[0] * n_gates / dt, dt, restored


def other_configs(q, wl, dev, stream, names=("cfg3", "cfg4")):
    """The other large BASELINE configs on the same GPU (parity cases, not the
    headline): per call, the median of 5 CUDA-event timings after 2 warm-ups,
    algorithmic GB/s and the fraction of the measured copy bandwidth."""
    import torch
    hbm, _ = peaks()
    out = {}
    for name in names:
        cfg = wl.CONFIGS[name]
        g, M, N = cfg.gates(), cfg.M, cfg.N
        e = 8 if cfg.dtype == "c64" else 16
        k1 = torch.empty(N * e, dtype=torch.uint8, device=dev)
        scale = cfg.state.scale() if M <= 30 else None
        stage = torch.empty(min(N, 1 << 26) * e, dtype=torch.uint8, pin_memory=True)
        for s0 in range(0, N, 1 << 26):
            c = min(N - s0, 1 << 26)
            wl.fill_state(cfg.state, stage.data_ptr(), s0, c, scale=scale)
            k1[s0 * e:(s0 + c) * e].copy_(stage[:c * e])
        del stage
        k2 = torch.empty_like(k1)
        perm = torch.empty(N, dtype=torch.int32, device=dev)
        ws = q.workspace(dev)
        plan = q.plan_create(g, M, cfg.dtype)
        torch.cuda.synchronize()
        if not (plan.flags & 1):
            q.plan_tune(plan, g, perm, k1, k2, ws, stream=stream)
        q.build_map(g, M, perm, stream=stream)
        calls = {
            "map_gather_planned": (lambda: q.map_gather_planned(plan, g, perm, k1, k2, ws, stream=stream),
                                   4 + 2 * e),
            "run_fused_planned": (lambda: q.run_fused_planned(plan, g, k1, k2, ws, stream=stream), 2 * e),
            "apply_map_planned": (lambda: q.apply_map_planned(plan, perm, k1, k2, ws, stream=stream),
                                  4 + 2 * e),
        }
        res = {"M": M, "dtype": cfg.dtype, "natural_order_plan": bool(plan.flags & 1)}
        for call, (f, bpe) in calls.items():
            ts = []
            for i in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    a.record(stream)
                    f()
                    b.record(stream)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            gbps = N * bpe / (ms * 1e-3) / 1e9
            res[call] = {"ms": ms, "entries_per_s": N / (ms * 1e-3), "GBps": gbps,
                         "bytes_per_entry": bpe, "frac_of_peak": gbps / hbm, "kernel": q.last_kernel()}
        out[name] = res
        del k1, k2, perm, calls
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------- main arm
def run_qsim(args):
    import torch
    import paper_quant_ph_0308158_b200 as q
    import workloads as wl

    world, rank, local = dist_setup()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    cfg = wl.CONFIGS[args.config]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    e = 8 if cfg.dtype == "c64" else 16
    stream = torch.cuda.Stream(dev)

    # ---- inputs: seeded on the host (pinned), copied once to HBM
    t_setup = time.perf_counter()
    def host_buffer(nbytes):
        """Pinned host memory, else pageable (e.g. 8 ranks x 64 GiB pinned may not fit)."""
        try:
            return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True), "pinned"
        except RuntimeError:
            return torch.empty(nbytes, dtype=torch.uint8), "pageable"

    # full host copies of the state (e2e input/output, CPU baseline) only when
    # every rank on this node fits them in host memory; else fill HBM through a
    # 1 GiB staging buffer and skip the e2e leg (recorded)
    import psutil
    need = world * 2 * N * e + (32 << 30)
    host_ok = psutil.virtual_memory().available >= need
    if os.environ.get("QSIM_BENCH_LOW_HOST_MEM") == "1":  # exercise the low-memory setup
        host_ok = False
    k1 = torch.empty(N * e, dtype=torch.uint8, device=dev)
    if host_ok:
        k1_host, k1_host_kind = host_buffer(N * e)
        wl.fill_state(cfg.state, k1_host.data_ptr())
        k1.copy_(k1_host, non_blocking=True)
    else:
        k1_host, k1_host_kind = None, "none"
        chunk = min(N, (1 << 30) // e)
        stage = torch.empty(chunk * e, dtype=torch.uint8, pin_memory=True)
        scale = cfg.state.scale()
        for s0 in range(0, N, chunk):
            wl.fill_state(cfg.state, stage.data_ptr(), s0, chunk, scale=scale)
            k1[s0 * e:(s0 + chunk) * e].copy_(stage)
        del stage
    perm = torch.empty(N, dtype=torch.int32, device=dev)
    k2 = torch.empty(N * e, dtype=torch.uint8, device=dev)
    ws = q.workspace(dev)
    t_plan = time.perf_counter()
    plan = q.plan_create(gates, M, cfg.dtype)      # host analysis, once per circuit
    t_plan = time.perf_counter() - t_plan
    # measured plan (like an FFTW_MEASURE plan): variants timed on these buffers,
    # the fastest map + gather kept; once per circuit, outside the timed region
    t_tune = time.perf_counter()
    torch.cuda.synchronize()                     # k1's H2D copy (default stream) is complete
    tuned = q.plan_tune(plan, gates, perm, k1, k2, ws, stream=stream) if not (plan.flags & 1) else -1
    t_tune = time.perf_counter() - t_tune
    # the planned apply (two-call mode) gets its own measured order: it reads
    # perm in plan order instead of writing it (all stages, about 60 s)
    t_tune_ap = time.perf_counter()
    plan_ap = q.plan_create(gates, M, cfg.dtype)
    if not (plan_ap.flags & 1):
        q.plan_tune(plan_ap, gates, perm, k1, k2, ws, stream=stream,
                    effort=q.TUNE_PATIENT | q.TUNE_APPLY)
    t_tune_ap = time.perf_counter() - t_tune_ap
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup

    from paper_quant_ph_0308158_b200.dist import barrier, max_over_ranks

    def timed_loop(step_fn, steps, warmup, per_kernel=None, name="step"):
        for _ in range(warmup):
            step_fn(None)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        marks = [] if per_kernel else None
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        launches = 0
        # an NVTX range around the timed launches: the ncu launch list and the
        # full capture of the step select them with --nvtx-include "timed_<name>/"
        torch.cuda.nvtx.range_push(f"timed_{name}")
        with torch.cuda.stream(stream):
            t0.record(stream)
            for _ in range(steps):
                launches += step_fn(marks)
            t1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ms = max_over_ranks(t0.elapsed_time(t1), device=dev)
        kern = {}
        if marks:
            for name, a, b in marks:
                kern.setdefault(name, []).append(a.elapsed_time(b))
        return ms, launches, kern

    def ev():
        x = torch.cuda.Event(enable_timing=True)
        x.record(stream)
        return x

    def step_materialised(marks):
        with torch.cuda.stream(stream):
            a = ev() if marks is not None else None
            q.build_map(gates, M, perm, stream=stream)
            n = q.last_launch_count()
            b = ev() if marks is not None else None
            q.apply_map_planned(plan_ap, perm, k1, k2, ws, stream=stream)
            n += q.last_launch_count()
            c = ev() if marks is not None else None
            if marks is not None:
                marks.append(("build_map", a, b))
                marks.append(("apply_map", b, c))
        return n

    def step_map_gather(marks):
        with torch.cuda.stream(stream):
            a = ev() if marks is not None else None
            q.map_gather_planned(plan, gates, perm, k1, k2, ws, stream=stream)
            n = q.last_launch_count()
            b = ev() if marks is not None else None
            if marks is not None:
                marks.append(("map_gather", a, b))
        return n

    qubits = wl.random_qubits(M, 2024, cfg.dtype)

    def step_kron(marks):
        with torch.cuda.stream(stream):
            a = ev() if marks is not None else None
            q.run_fused_kron(gates, M, qubits, k2, dtype=cfg.dtype, stream=stream)
            n = q.last_launch_count()
            b = ev() if marks is not None else None
            if marks is not None:
                marks.append(("fused_kron", a, b))
        return n

    # M = 40 (beyond a stored state): a 2^M-entry portion of a 40-qubit
    # circuit's output with the input generated on the fly (64-bit walk)
    M40 = 40
    gates40 = wl.random_gates(64, M40, 4)
    qubits40 = wl.random_qubits(M40, 2040, cfg.dtype)
    start40 = (1 << (M40 - 1)) - N // 2          # straddles the middle of the 2^40 outputs

    def step_kron40(marks):
        with torch.cuda.stream(stream):
            a = ev() if marks is not None else None
            q.run_fused_kron(gates40, M40, qubits40, k2, start=start40, count=N, dtype=cfg.dtype,
                             stream=stream)
            n = q.last_launch_count()
            b = ev() if marks is not None else None
            if marks is not None:
                marks.append(("fused_kron40", a, b))
        return n

    def step_fused(marks):
        with torch.cuda.stream(stream):
            a = ev() if marks is not None else None
            q.run_fused_planned(plan, gates, k1, k2, ws, stream=stream)
            n = q.last_launch_count()
            b = ev() if marks is not None else None
            if marks is not None:
                marks.append(("run_fused", a, b))
        return n

    def step_plain_fused(marks):
        with torch.cuda.stream(stream):
            a = ev() if marks is not None else None
            q.run_fused(gates, M, k1, k2, stream=stream, dtype=cfg.dtype)
            n = q.last_launch_count()
            b = ev() if marks is not None else None
            if marks is not None:
                marks.append(("plain_run_fused", a, b))
        return n

    def step_plain_apply(marks):
        with torch.cuda.stream(stream):
            a = ev() if marks is not None else None
            q.apply_map(perm, M, k1, k2, stream=stream, dtype=cfg.dtype)
            n = q.last_launch_count()
            b = ev() if marks is not None else None
            if marks is not None:
                marks.append(("plain_apply_map", a, b))
        return n

    sampler = ClockSampler(local)
    with sampler:
        ms_mg, launches_mg, kern_mg = timed_loop(step_map_gather, args.steps, args.warmup,
                                                 per_kernel=True, name="map_gather")
        kern_name_mg = q.last_kernel()
        # the timed step's own output, checked against the oracle before any
        # other loop overwrites perm / k2
        verified = verify_sample(gates, M, e, perm, k2, k1_host, cfg, dev)
        ms_mat, launches_mat, kern_mat = timed_loop(step_materialised, args.steps, args.warmup,
                                                    per_kernel=True, name="materialised")
        ms_fused, launches_fused, kern_fused = timed_loop(step_fused, args.steps, args.warmup,
                                                          per_kernel=True, name="fused")
        plain_steps = max(2, args.steps // 4)
        ms_pf, launches_pf, kern_pf = timed_loop(step_plain_fused, plain_steps, args.warmup,
                                                 per_kernel=True, name="plain_fused")
        kern_name_pf = q.last_kernel()
        q.build_map(gates, M, perm, stream=stream)
        ms_pa, launches_pa, kern_pa = timed_loop(step_plain_apply, plain_steps, min(args.warmup, 1),
                                                 per_kernel=True, name="plain_apply")
        ms_kron, launches_kron, kern_kron = timed_loop(step_kron, args.steps, args.warmup,
                                                       per_kernel=True, name="kron")
        kern_name_kron = q.last_kernel()
        ms_k40, launches_k40, kern_k40 = timed_loop(step_kron40, max(2, args.steps // 4),
                                                    args.warmup, per_kernel=True, name="kron40")
        kern_name_k40 = q.last_kernel()
        # write-only ceiling for the on-the-fly input's roofline: torch's fill
        # of the same 2^M-entry output buffer (not our kernel; a denominator)
        wz = []
        for _ in range(4):
            a0, b0 = ev(), ev()
            a0.record(stream)
            with torch.cuda.stream(stream):
                k2.view(torch.float32).zero_()
            b0.record(stream)
            b0.synchronize()
            wz.append(a0.elapsed_time(b0))
        write_peak = N * e / (min(wz[1:]) * 1e-3) / 1e9
    clocks = sampler.summary()

    # ---- launch-bound small state (cfg2, 2^20 entries, L2-resident): the
    # planned step called directly vs replayed from a CUDA graph
    launch_bound = None
    if rank == 0:
        c2 = wl.CONFIGS["cfg2"]
        g2, n2 = c2.gates(), c2.N
        a2 = torch.zeros(n2 * 8, dtype=torch.uint8, device=dev)
        b2 = torch.empty_like(a2)
        p2 = torch.empty(n2, dtype=torch.int32, device=dev)
        plan2 = q.plan_create(g2, c2.M, c2.dtype)
        reps = 100

        def direct():
            for _ in range(reps):
                q.map_gather_planned(plan2, g2, p2, a2, b2, ws, stream=stream)
        graph = q.Graph(plan2, g2, q.GRAPH_MAP_GATHER, p2, a2, b2, ws, reps=reps)

        def replay():
            graph.launch(stream=stream)
        res = {}
        for name, fn in (("direct", direct), ("graph", replay)):
            with torch.cuda.stream(stream):
                fn()
                torch.cuda.synchronize()
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record(stream)
                fn()
                t1.record(stream)
            torch.cuda.synchronize()
            res[name] = 1e3 * t0.elapsed_time(t1) / reps
        graph.close()
        # warm (back to back, the 20 MiB working set stays in L2) vs flushed
        # (a 256 MiB scrub written between steps evicts it)
        scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        warm, flushed = [], []
        for _ in range(12):
            for lst, flush in ((warm, False), (flushed, True)):
                with torch.cuda.stream(stream):
                    if flush:
                        scrub.fill_(1)
                    # keep the GPU busy while the call is enqueued, so the events
                    # bracket the kernel and not the host's launch latency
                    torch.cuda._sleep(100000)
                    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    t0.record(stream)
                    q.map_gather_planned(plan2, g2, p2, a2, b2, ws, stream=stream)
                    t1.record(stream)
                torch.cuda.synchronize()
                lst.append(t0.elapsed_time(t1))
        del scrub
        launch_bound = {"config": "cfg2 (M = 20, 2^20 entries, L2-resident)",
                        "call": "qsim_map_gather_planned", "direct_us_per_step": res["direct"],
                        "graph_us_per_step": res["graph"],
                        "warm_us": 1e3 * statistics.median(warm[2:]),
                        "flushed_us": 1e3 * statistics.median(flushed[2:]),
                        "kernel": q.last_kernel(),
                        "note": "CUDA graph of 100 recorded steps (qsim_graph_*) vs 100 calls; "
                                "warm = back to back (L2-resident), flushed = 256 MiB written "
                                "between steps; one call each, CUDA events around the kernel "
                                "(a GPU sleep before the start event hides the launch latency)"}
        del a2, b2, p2

    # ---- end to end through the C ABI from pinned host buffers: every step
    # copies its input in and its result out; qsim_run_host_batch overlaps
    # step i+1's copy in and step i-1's copy out with step i's compute
    # (double-buffered device state)
    e2e = None
    if not host_ok and not args.no_e2e:
        e2e = {"skipped": f"host memory: {world} ranks x 2 x {N * e >> 30} GiB state copies "
                          f"do not fit ({psutil.virtual_memory().available >> 30} GiB available)"}
    elif not args.no_e2e and args.e2e_steps > 0:
        k2_host, k2_host_kind = host_buffer(N * e)
        k1b = torch.empty(N * e, dtype=torch.uint8, device=dev)
        k2b = torch.empty(N * e, dtype=torch.uint8, device=dev)
        ns = args.e2e_steps
        q.run_host_batch(gates, M, q.MATERIALISED, [k1_host], [k2_host], [k1, k1b], [k2, k2b], perm,
                         ws, dtype=cfg.dtype)                     # warm-up (plan + JIT cached)
        barrier()
        t0 = time.perf_counter()
        q.run_host_batch(gates, M, q.MATERIALISED, [k1_host] * ns, [k2_host] * ns, [k1, k1b],
                         [k2, k2b], perm, ws, dtype=cfg.dtype)
        dt = max_over_ranks(time.perf_counter() - t0, device=dev)
        e2e = {"value": world * N * ns / dt, "unit": "entries/s",
               "h2d_bytes_per_step": N * e, "d2h_bytes_per_step": N * e,
               "ms_per_step": 1e3 * dt / ns, "steps": ns,
               "host_memory": f"k1 {k1_host_kind}, k2 {k2_host_kind}",
               "path": "qsim_run_host_batch: per step H2D k1 (pinned) -> map_gather (perm + k2) -> "
                       "D2H k2, copies overlapped with compute across steps, synchronised at the end"}
        # the unpipelined single call, for reference
        t0 = time.perf_counter()
        q.run_host(gates, M, q.MATERIALISED, k1_host, k2_host, k1, k2, perm, ws,
                   stream=stream, dtype=cfg.dtype)
        e2e["single_call_ms"] = 1e3 * (time.perf_counter() - t0)
        del k2_host, k1b, k2b
        torch.cuda.empty_cache()

    # ---- the other large configs (rank 0): cfg3 (well-mixed) and cfg4 (ripple)
    others = None
    if rank == 0 and args.config == "cfg5" and not args.no_other_configs:
        others = other_configs(q, wl, dev, stream)

    # ---- cpu baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and k1_host is not None:
        import workloads as wl2
        k1_np = k1_host.numpy().view(wl2.NP_DTYPE[cfg.dtype])
        threads = len(os.sched_getaffinity(0))
        count = min(N, 1 << args.cpu_sample_log2)
        rate, dt = cpu_oracle_rate(gates, k1_np, 0, count, threads)
        c1 = min(N, 1 << 24)
        rate1, dt1, core = cpu_single_core(gates, k1_np, c1)
        acc_rate, acc_dt, restored = cpu_accumulate(gates, k1_np, 1)
        cpu = {"value": rate, "unit": "entries/s", "cores": threads, "kind": "oracle",
               "seconds": dt,
               "sample": f"output entries [0, 2^{args.cpu_sample_log2}) of {args.config} "
                         f"(build_map walk + apply gather, oracle C -O2, one thread per core "
                         f"on disjoint sub-ranges)",
               "single_core": {"value": rate1, "unit": "entries/s", "cores": 1, "core": core,
                               "seconds": dt1,
                               "sample": f"output entries [0, 2^{c1.bit_length() - 1}) of "
                                         f"{args.config}, build walk + apply gather, process "
                                         f"pinned to one core (taskset -c {core} equivalent)",
                               "projected_full_s": N / rate1},
               "accumulate": {"value": acc_rate, "unit": "entry-steps/s", "cores": 1,
                              "seconds": acc_dt, "k1_restored": restored,
                              "sample": f"the paper's basic accumulation method (P:L59), step 1 of "
                                        f"{args.config} over all 2^{M} entries, one core",
                              "projected_full_s": N * int(gates.shape[0]) / acc_rate},
               **host_info()}

    if rank != 0:
        return
    hbm, hbm_src = peaks()
    bytes_apply = N * (4 + 2 * e)          # read perm, gather k1, write k2
    bytes_build = N * 4                    # write perm
    bytes_fused = N * 2 * e                # gather k1, write k2
    bytes_mg = N * (4 + 2 * e)             # write perm, gather k1, write k2
    mg_ms = statistics.mean(kern_mg["map_gather"])
    apply_ms = statistics.mean(kern_mat["apply_map"])
    build_ms = statistics.mean(kern_mat["build_map"])
    fused_ms = statistics.mean(kern_fused["run_fused"])
    kron_ms = statistics.mean(kern_kron["fused_kron"])
    k40_ms = statistics.mean(kern_k40["fused_kron40"])
    ms_step = ms_mg / args.steps
    achieved = bytes_mg / (mg_ms * 1e-3) / 1e9
    split = bool(plan.flags & q.PLAN_SPLIT)
    if split:
        mg_kernel = (f"{kern_name_mg}: the planned gather (NVRTC, circuit-specialised, k2 only) "
                     "then the natural-order build (perm), two launches per step")
    else:
        mg_kernel = (f"{kern_name_mg} (NVRTC, circuit-specialised, perm + gather, one launch)"
                     if launches_mg == args.steps else f"{kern_name_mg} (no JIT)")

    def gbps(b, ms):
        return b / (ms * 1e-3) / 1e9

    line = {
        "metric": METRIC,
        "value": world * N / (ms_step * 1e-3),
        "unit": "entries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded counter-based Gaussian state, numpy PCG64 gate list)",
        "config": {"workload": f"{args.config}: {cfg.description}", "M": M,
                   "n_gates": int(gates.shape[0]), "state_dtype": "complex64" if e == 8 else
                   "complex128",
                   "step": "qsim_map_gather_planned: materialised map (perm, uint32) + gather "
                           "k2 = k1[perm]" + (" -- two kernels (plan flag QSIM_PLAN_SPLIT: "
                                              "planned gather, then natural-order build)"
                                              if split else ", one kernel"),
                   "l2": "inputs larger than L2 (k1, k2 %d GiB each; perm %d GiB)"
                   % (N * e >> 30, N * 4 >> 30), "parallelism": f"replicas x{world}"},
        "achieved_GBps": gbps(bytes_mg, ms_step),
        "frac_of_8TBps": gbps(bytes_mg, ms_step) * 1e9 / 8e12,
        "roofline": {"bound": "hbm", "kernel": mg_kernel, "achieved": achieved,
                     "peak": hbm, "peak_source": hbm_src, "unit": "GB/s",
                     "frac": achieved / hbm, "frac_of_8TBps": achieved * 1e9 / 8e12,
                     "traffic": ncu_traffic(args.config, "map_gather_split" if split
                                            else "map_gather"),
                     "scope": ("the step's two launches together (the call's CUDA-event "
                               "duration); per launch in per_kernel" if split else
                               "the step's one launch"),
                     "per_kernel": ({
                         "gather": {"kernel": "qsim_jit_fused (same plan, same kernel instance as "
                                              "modes.run_fused)", "ms": fused_ms,
                                    "bytes_per_entry": 2 * e, "GBps": gbps(bytes_fused, fused_ms),
                                    "frac": gbps(bytes_fused, fused_ms) / hbm},
                         "build": {"kernel": "qsim_jit_build (natural order, as modes.build_map)",
                                   "ms": build_ms, "bytes_per_entry": 4,
                                   "GBps": gbps(bytes_build, build_ms),
                                   "frac": gbps(bytes_build, build_ms) / hbm}} if split else None),
                     "algorithmic_bytes_per_launch": bytes_mg,
                     "algorithmic_bytes_per_entry": 4 + 2 * e,
                     "note": "DRAM traffic ~1.04x algorithmic (ncu); bound: the random k1 reads, "
                             "fetched by L2 as separate 32-B sectors unless a line's sectors share "
                             "one warp instruction (DESIGN.md section 6, profiles/r01_mb_window.jsonl)"},
        "modes": {
            "map_gather": {"ms": mg_ms, "GBps": achieved, "entries_per_s": N / (mg_ms * 1e-3),
                           "launches_per_step": launches_mg / args.steps,
                           "form": ("two kernels: planned gather, natural-order build (QSIM_PLAN_SPLIT)"
                                    if split else "one kernel: perm stored in plan order + gather"),
                           "kernel": kern_name_mg},
            "two_call": {"ms": ms_mat / args.steps, "entries_per_s": N / (ms_mat / args.steps * 1e-3),
                         "calls": "qsim_build_map + qsim_apply_map_planned"},
            "build_map": {"ms": build_ms, "GBps": gbps(bytes_build, build_ms),
                          "entries_per_s": N / (build_ms * 1e-3), "bytes_per_entry": 4,
                          "frac_of_peak": gbps(bytes_build, build_ms) / hbm},
            "apply_map": {"ms": apply_ms, "GBps": gbps(bytes_apply, apply_ms),
                          "entries_per_s": N / (apply_ms * 1e-3), "bytes_per_entry": 4 + 2 * e,
                          "frac_of_peak": gbps(bytes_apply, apply_ms) / hbm},
            "run_fused": {"ms": fused_ms, "GBps": gbps(bytes_fused, fused_ms),
                          "entries_per_s": N / (fused_ms * 1e-3), "bytes_per_entry": 2 * e,
                          "frac_of_peak": gbps(bytes_fused, fused_ms) / hbm},
            "plain_run_fused": {
                "ms": statistics.mean(kern_pf["plain_run_fused"]),
                "entries_per_s": N / (statistics.mean(kern_pf["plain_run_fused"]) * 1e-3),
                "GBps": gbps(bytes_fused, statistics.mean(kern_pf["plain_run_fused"])),
                "kernel": kern_name_pf,
                "note": "qsim_run_fused (north-star call, no plan argument): plans internally, "
                        "plan cached per circuit, round-robin chunks (no workspace)"},
            "plain_apply_map": {
                "ms": statistics.mean(kern_pa["plain_apply_map"]),
                "entries_per_s": N / (statistics.mean(kern_pa["plain_apply_map"]) * 1e-3),
                "GBps": gbps(bytes_apply, statistics.mean(kern_pa["plain_apply_map"])),
                "note": "qsim_apply_map (north-star call): natural output order, k_apply; it "
                        "receives no gates, so it cannot plan -- the fast form of the same "
                        "call is qsim_apply_map_planned (modes.apply_map)"},
            "fused_kron": {"ms": kron_ms, "GBps": gbps(N * e, kron_ms),
                           "entries_per_s": N / (kron_ms * 1e-3), "bytes_per_entry": e,
                           "frac_of_peak": gbps(N * e, kron_ms) / hbm,
                           "frac_of_write_peak": gbps(N * e, kron_ms) / write_peak,
                           "kernel": kern_name_kron,
                           "note": "qsim_run_fused_kron: Appendix-1 input generated on the fly "
                                   "(k1 never read), write-only"},
            "fused_kron_M40_portion": {
                "ms": k40_ms, "GBps": gbps(N * e, k40_ms), "entries_per_s": N / (k40_ms * 1e-3),
                "bytes_per_entry": e, "frac_of_peak": gbps(N * e, k40_ms) / hbm,
                "frac_of_write_peak": gbps(N * e, k40_ms) / write_peak, "kernel": kern_name_k40,
                "note": "M = 40 qubits (64 random gates, seed 4): output portion "
                        "[2^39 - 2^31, 2^39 + 2^31) of 2^40, input on the fly, 64-bit walk"},
        },
        "write_peak": {"GBps": write_peak, "how": "torch zero_ of the 2^M-entry output buffer, "
                                                 "best of 3 (write-only roofline of fused_kron)"},
        "launch_bound": launch_bound,
        "verified": verified,
        "other_configs": others,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_mg,
        "gpu_launches_other_loops": {"two_call": launches_mat, "fused": launches_fused,
                                     "plain_run_fused": launches_pf, "plain_apply_map": launches_pa,
                                     "fused_kron": launches_kron, "fused_kron_M40": launches_k40},
        "clocks": clocks,
        "setup_s": t_setup,
        "jit": {"status": q.jit_status(), "last_compile_ms": q.jit_last_compile_ms(),
                "note": "kernels NVRTC-compiled for the circuit on first use (warm-up steps); "
                        "timed steps reuse them"},
        "plan_apply": {"tune_seconds": t_tune_ap, "sigma": list(plan_ap.sigma)[:M],
                       "chunk_log2": plan_ap.chunk_log2, "blocks_per_sm": plan_ap.blocks_per_sm,
                       "note": "the two-call mode's qsim_apply_map_planned uses its own plan, "
                               "qsim_plan_tune_ex(QSIM_TUNE_PATIENT | QSIM_TUNE_APPLY)"},
        "plan": {"seconds": t_plan, "tune_seconds": t_tune, "tuned_variant": tuned,
                 "sigma": list(plan.sigma)[:M], "chunk_log2": plan.chunk_log2,
                 "fused_chunk_log2": plan.fused_chunk_log2, "blocks_per_sm": plan.blocks_per_sm,
                 "natural_order": bool(plan.flags & 1), "split": split,
                 "cta_threads": plan.cta_threads, "flags": plan.flags,
                 "sector_cover_bits": plan.tile_log2,
                 "sector_pairs_contained": plan.tile_contained,
                 "note": "qsim_plan_create (host sampling of the circuit) and qsim_plan_tune "
                         "(measured variants) run once per circuit, outside the timed region, "
                         "like an FFTW_MEASURE plan"},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ reference arm
def run_reference(args):
    """The oracle (this tier's reference arm), timed on the host cores."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    import workloads as wl
    cfg = wl.CONFIGS[args.config]
    gates, N = cfg.gates(), cfg.N
    k1 = np.empty(N, dtype=wl.NP_DTYPE[cfg.dtype])
    wl.fill_state(cfg.state, k1.ctypes.data)
    threads = os.cpu_count() or 1
    count = min(N, 1 << 26)           # bounded sample per step
    for _ in range(args.warmup):
        cpu_oracle_rate(gates, k1, 0, min(count, 1 << 20), threads)
    times = []
    for s in range(args.steps):
        start = (s * count) % N
        _, dt = cpu_oracle_rate(gates, k1, start, count, threads)
        times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = count / (ms * 1e-3)
    sample = (f"each step: {count} consecutive outputs of {args.config} (of 2^{cfg.M}); "
              f"oracle build walk + apply gather, one thread per core")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "entries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": {"workload": f"{args.config}: {cfg.description}",
                                              "M": cfg.M, "n_gates": int(gates.shape[0])},
            "cpu_baseline": {"value": value, "unit": "entries/s", "cores": threads,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_qsim(a)
