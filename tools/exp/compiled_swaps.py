"""Experiment: exchanges that touch the compiled part of the traversal order
(counter positions 0..9: lanes and in-thread entries; each new order is a
new NVRTC kernel), screened on cfg5 map+gather from the stage-4 tuned plan."""
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
cfg = wl.CONFIGS["cfg5"]
gates, M, N = cfg.gates(), cfg.M, cfg.N
k1 = torch.empty(N * 8, dtype=torch.uint8, device=dev)
stage = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
chunk = (1 << 30) // 8
scale = cfg.state.scale()
for s0 in range(0, N, chunk):
    wl.fill_state(cfg.state, stage.data_ptr(), s0, chunk, scale=scale)
    k1[s0 * 8:(s0 + chunk) * 8].copy_(stage)
del stage
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device=dev)
ws = q.workspace(dev)
plan = q.plan_create(gates, M, "c64")
rec = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_plan_cfg5_stage4.json")))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(sig, reps):
    for k in range(32):
        plan.sigma[k] = sig[k]
    plan.chunk_log2 = plan.fused_chunk_log2 = rec["chunk_log2"]
    q.map_gather_planned(plan, gates, perm, k1, k2, ws)  # compiles a new order
    best = 1e30
    for _ in range(reps):
        a.record()
        q.map_gather_planned(plan, gates, perm, k1, k2, ws)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


base = [int(x) for x in os.environ["CS_BASE"].split(",")] if os.environ.get("CS_BASE") else list(rec["sigma"])
base_t = t(base, 5)
print(json.dumps({"base_ms": base_t, "sigma": base}), flush=True)
t0 = time.time()
scr = []
for i in range(3, 10):  # positions 0..2 stay output bits 0..2 (plan_keep_bits)
    for j in range(i + 1, 32):
        s = list(base)
        s[i], s[j] = s[j], s[i]
        scr.append((t(s, 1), i, j, s))
scr.sort()
print(json.dumps({"screened": len(scr), "seconds": time.time() - t0,
                  "top8": [(round(x[0], 3), x[1], x[2]) for x in scr[:8]],
                  "worst": round(scr[-1][0], 2)}), flush=True)
for x in scr[:6]:
    ab = [(t(base, 3), t(x[3], 3)) for _ in range(3)]
    print(json.dumps({"swap": [x[1], x[2]], "base_ms": min(p[0] for p in ab), "cand_ms": min(p[1] for p in ab),
                      "sigma": x[3]}), flush=True)
