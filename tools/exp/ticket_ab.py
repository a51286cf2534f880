"""Experiment (sustained) -- chunk-ticket prefetch A/B.  AB_SWITCH names the
generated-source switch (QSIM_TICKET_AHEAD, QSIM_TILE_DYN, QSIM_GATHER_PIPE);
each existed only in its experiment build. QSIM_TICKET_AHEAD (a generated-source
macro, now fixed: on for the gathers, off for the apply); result in
profiles/r02_ticket_ahead_ab.json.  (Header of split_sustained.py follows.) cfg5 map + gather as one kernel (perm stored in plan order) vs
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

a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
STEPS = int(os.environ.get("SC_STEPS", "20"))
SWITCH = os.environ.get("AB_SWITCH", "QSIM_TICKET_AHEAD")   # a generated-source A/B switch
calls = {
    "map_gather": lambda: q.map_gather_planned(plan, gates, perm, k1, k2, ws),
    "fused": lambda: q.run_fused_planned(plan, gates, k1, k2, ws),
    "apply": lambda: q.apply_map_planned(plan, perm, k1, k2, ws),
}


def loop(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(STEPS):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / STEPS


ok = {}
for mode in ("0", "1"):                      # compile both variants, check bytes
    os.environ[SWITCH] = mode
    perm.fill_(-1)
    k2.fill_(0)
    calls["map_gather"]()
    torch.cuda.synchronize()
    ok[mode] = bool(torch.equal(perm, ref_perm) and torch.equal(k2, ref_k2))
res = {f"{c}/{SWITCH}={m}": [] for c in calls for m in ("0", "1")}
for _ in range(int(os.environ.get("SC_REPS", "4"))):
    for c, fn in calls.items():
        for m in ("0", "1"):
            os.environ[SWITCH] = m
            res[f"{c}/{SWITCH}={m}"].append(loop(fn))
print(json.dumps({"variant": variant, "flags": plan.flags, "bytes_equal": ok, "steps_per_loop": STEPS,
                  "ms_per_step_each_loop": res,
                  "ms_mean": {n: sum(v) / len(v) for n, v in res.items()}}))
