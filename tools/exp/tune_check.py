"""Run qsim_plan_tune on cfg5 (the bench's Gaussian state) and time the kept
plan against the recorded round-2 plan (interleaved, best of 3 x 5)."""
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
t0 = time.time()
variant = q.plan_tune(plan, gates, perm, k1, k2, ws)
tune_s = time.time() - t0
old = q.plan_create(gates, M, "c64")
rec = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_plan_cfg5.json")))
for k, v in enumerate(rec["sigma"]):
    old.sigma[k] = v
old.chunk_log2, old.fused_chunk_log2 = rec["chunk_log2"], rec["fused_chunk_log2"]
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(p):
    best = 1e30
    for _ in range(3):
        a.record()
        q.map_gather_planned(p, gates, perm, k1, k2, ws)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


sw = q.plan_create(gates, M, "c64")
ctypes_copy = bytes(plan)
import ctypes  # noqa: E402
ctypes.memmove(ctypes.addressof(sw), ctypes_copy, len(ctypes_copy))
i, j = [int(x) for x in os.environ.get("TC_SWAP", "3,6").split(",")]
sw.sigma[i], sw.sigma[j] = plan.sigma[j], plan.sigma[i]
res = {"new": [], "recorded": [], "swapped": []}
for _ in range(5):
    res["new"].append(t(plan))
    res["recorded"].append(t(old))
    res["swapped"].append(t(sw))
print(json.dumps({"tune_s": tune_s, "variant": variant, "sigma": list(plan.sigma),
                  "chunk_log2": plan.chunk_log2, "new_ms": min(res["new"]),
                  "recorded_ms": min(res["recorded"]), "swapped_ms": min(res["swapped"]),
                  "swapped_sigma": list(sw.sigma), "all": res}), flush=True)
