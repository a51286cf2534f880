"""Steady-state time of every planned call on every BASELINE config (CUDA events, median of 5 after 2
warm-ups); one JSON line per (config, call)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
    cfg = wl.CONFIGS[name]
    g, M, N = cfg.gates(), cfg.M, cfg.N
    e = 8 if cfg.dtype == "c64" else 16
    k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
    torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
    k2 = torch.empty_like(k1)
    perm = torch.empty(N, dtype=torch.int32, device="cuda")
    ws = q.workspace()
    plan = q.plan_create(g, M, cfg.dtype)
    calls = {
        "build_map": (lambda: q.build_map(g, M, perm), 4),
        "apply_map_planned": (lambda: q.apply_map_planned(plan, perm, k1, k2, ws), 4 + 2 * e),
        "run_fused_planned": (lambda: q.run_fused_planned(plan, g, k1, k2, ws), 2 * e),
        "map_gather_planned": (lambda: q.map_gather_planned(plan, g, perm, k1, k2, ws), 4 + 2 * e),
    }
    for call, (fn, bpe) in calls.items():
        ms = timeit(fn)
        print(json.dumps({"config": name, "M": M, "dtype": cfg.dtype, "call": call,
                          "ms": round(ms, 4), "entries_per_s": N / ms * 1e3,
                          "GBps": N * bpe / ms / 1e6, "natural_order": bool(plan.flags & 1),
                          "kernel": q.last_kernel() or "natural/AOT"}), flush=True)
    del k1, k2, perm, calls
    torch.cuda.empty_cache()
