"""Experiment (sustained): the planned apply with the chunk ticket taken one chunk
ahead or not (QSIM_APPLY_AHEAD existed only in the experiment build), EACH with
the plan qsim_plan_tune_ex(PATIENT | APPLY) keeps for it.
Result: profiles/r02_apply_ahead_ab.json."""
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
cfg = wl.CONFIGS[os.environ.get("SC_CONFIG", "cfg5")]
gates, M, N = cfg.gates(), cfg.M, cfg.N
e = 8 if cfg.dtype == "c64" else 16
k1 = torch.empty(N * e, dtype=torch.uint8, device=dev)
stage = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
chunk = (1 << 30) // e
scale = cfg.state.scale()
for s0 in range(0, N, chunk):
    c = min(chunk, N - s0)
    wl.fill_state(cfg.state, stage.data_ptr(), s0, c, scale=scale)
    k1[s0 * e:(s0 + c) * e].copy_(stage[:c * e])
del stage
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device=dev)
ws = q.workspace(dev)
torch.cuda.synchronize()
plan = q.plan_create(gates, M, cfg.dtype)
t0 = time.time()
variant = -1
tune_s = time.time() - t0

plans = {}
for mode in ("0", "1"):
    os.environ["QSIM_APPLY_AHEAD"] = mode
    p = q.plan_create(gates, M, cfg.dtype)
    v = q.plan_tune(p, gates, perm, k1, k2, ws, effort=q.TUNE_PATIENT | q.TUNE_APPLY)
    plans[mode] = (p, v)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def loop(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 20


res = {}
for _ in range(4):
    for mode, (p, v) in plans.items():
        os.environ["QSIM_APPLY_AHEAD"] = mode
        res.setdefault(f"apply/ahead={mode}", []).append(
            loop(lambda: q.apply_map_planned(p, perm, k1, k2, ws)))
print(json.dumps({"plans": {m: {"variant": v, "flags": p.flags, "sigma": list(p.sigma)[:M]}
                            for m, (p, v) in plans.items()},
                  "ms_per_step_each_loop": res,
                  "ms_mean": {n: sum(x) / len(x) for n, x in res.items()}}))
