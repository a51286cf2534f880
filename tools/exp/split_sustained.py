"""Experiment (sustained): cfg5 map + gather as one kernel (perm stored in plan order) vs
two kernels (QSIM_PLAN_SPLIT: the planned gather, then the natural-order
build).  Tunes once (qsim_plan_tune, which now also times the split form in
its first stage), then times, interleaved (5 rounds, best of 3 each):
  tuned        the kept plan as kept
  toggled      the same order in the other map + gather form
  recorded     a one-kernel plan tuned before the split form existed
               (profiles/r02_tuned_plan_cfg5_s6.json, if present)
and checks that every form gives the same perm / k2 bytes."""
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
variant = q.plan_tune(plan, gates, perm, k1, k2, ws)
tune_s = time.time() - t0
ref_perm, ref_k2 = perm.clone(), k2.clone()

plans = {"tuned": plan}
# QSIM_PLAN_NATMAP (8) existed only in commit dd6f732 (measured slower, removed)
NATMAP = getattr(q, "PLAN_NATMAP", None)
forms = (("one_kernel", 0), ("split", q.PLAN_SPLIT)) + ((("natmap", NATMAP),) if NATMAP else ())
for nm, form in forms:
    o = q.Plan.from_buffer_copy(plan)
    o.flags = (o.flags & ~(q.PLAN_SPLIT | (NATMAP or 0))) | form
    plans[nm + "(same order)"] = o
rec_path = os.path.join(ROOT, "profiles", "r02_tuned_plan_cfg5_s6.json")
if cfg is wl.CONFIGS["cfg5"] and os.path.exists(rec_path):
    rec = json.load(open(rec_path))
    old = q.plan_create(gates, M, cfg.dtype)
    for k, v in enumerate(rec["sigma"]):
        old.sigma[k] = v
    old.chunk_log2, old.fused_chunk_log2 = rec["chunk_log2"], rec["fused_chunk_log2"]
    old.blocks_per_sm, old.flags = rec.get("blocks_per_sm", 1), rec.get("flags", 0)
    old.cta_threads = rec.get("cta_threads", 256)
    plans["recorded"] = old


a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
STEPS = int(os.environ.get("SC_STEPS", "20"))


def loop(p):
    """bench.py's regime: warm-up steps, then STEPS back-to-back timed steps."""
    for _ in range(3):
        q.map_gather_planned(p, gates, perm, k1, k2, ws)
    torch.cuda.synchronize()
    a.record()
    for _ in range(STEPS):
        q.map_gather_planned(p, gates, perm, k1, k2, ws)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / STEPS


def fused_loop(p):
    for _ in range(3):
        q.run_fused_planned(p, gates, k1, k2, ws)
    torch.cuda.synchronize()
    a.record()
    for _ in range(STEPS):
        q.run_fused_planned(p, gates, k1, k2, ws)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / STEPS


ok = {}
for name, p in plans.items():               # warm (compiles) + byte check against the tuner's result
    perm.fill_(-1)
    k2.fill_(0)
    q.map_gather_planned(p, gates, perm, k1, k2, ws)
    torch.cuda.synchronize()
    ok[name] = bool(torch.equal(perm, ref_perm) and torch.equal(k2, ref_k2))
res = {n: [] for n in plans}
res["fused(tuned)"] = []
for _ in range(int(os.environ.get("SC_REPS", "4"))):
    for n, p in plans.items():
        res[n].append(loop(p))
    res["fused(tuned)"].append(fused_loop(plan))
out = {"variant": variant, "tune_s": tune_s, "flags": plan.flags, "sigma": list(plan.sigma)[:M],
       "bytes_equal": ok, "steps_per_loop": STEPS, "ms_per_step_each_loop": res,
       "ms_mean": {n: sum(v) / len(v) for n, v in res.items()}}
print(json.dumps(out))
