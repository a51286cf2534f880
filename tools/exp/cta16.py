"""Experiment: the cfg5 map+gather kernel with 16 warps per CTA (plan
cta_threads 512: a round covers counter bits 0..13) against 8 warps, same
order (the bench's tuned plan), interleaved A/B; parity on samples."""
import json
import os
import sys

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
tuned = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_s5.json")))["plan"]
plans = {}
for thr in (256, 512):
    for cl in (14, 15, 16):
        p = q.plan_create(gates, M, "c64")
        for k, v in enumerate(tuned["sigma"]):
            p.sigma[k] = v
        p.chunk_log2 = p.fused_chunk_log2 = cl
        p.cta_threads = thr
        plans[(thr, cl)] = p
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(p, fn="mg"):
    best = 1e30
    for _ in range(3):
        a.record()
        if fn == "mg":
            q.map_gather_planned(p, gates, perm, k1, k2, ws)
        elif fn == "fused":
            q.run_fused_planned(p, gates, k1, k2, ws)
        else:
            q.apply_map_planned(p, perm, k1, k2, ws)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


for p in plans.values():
    t(p)
res = {str(k): [] for k in plans}
for _ in range(3):
    for k, p in plans.items():
        res[str(k)].append(t(p))
print(json.dumps({"map_gather_ms": {k: min(v) for k, v in res.items()}}), flush=True)
for fn in ("fused", "apply"):
    q.build_map(gates, M, perm)
    r = {str(k): min(t(p, fn) for _ in range(2)) for k, p in plans.items() if k[1] == 15}
    print(json.dumps({fn + "_ms": r}), flush=True)
# parity of the 16-warp kernel on samples against a natural-order build
q.map_gather_planned(plans[(512, 15)], gates, perm, k1, k2, ws)
ref = torch.empty_like(perm)
q.build_map(gates, M, ref)
torch.cuda.synchronize()
idx = torch.randint(0, N, (1 << 22,), device=dev)
ok_p = bool(torch.equal(perm[idx], ref[idx]))
k2v, k1v = k2.view(torch.int64), k1.view(torch.int64)
ok_k = bool(torch.equal(k2v[idx], k1v[ref[idx].long() & 0xffffffff]))
print(json.dumps({"perm_ok": ok_p, "k2_ok": ok_k}), flush=True)
