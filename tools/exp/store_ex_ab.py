"""A/B (experiment): the exchanged store layout of the NVRTC gather kernels
(QSIM_STORE_EX=1, default) vs the plan's lane layout for the stores too
(QSIM_STORE_EX=0), for the recorded cfg5 plans; run once per setting."""
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
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
plans = {}
for name, f in (("s5", "r02_bench_s5.json"), ("s6", "r02_bench_s6.json")):
    p = q.plan_create(gates, M, "c64")
    for k, v in enumerate(json.load(open(os.path.join(ROOT, "profiles", f)))["plan"]["sigma"]):
        p.sigma[k] = v
    p.chunk_log2 = p.fused_chunk_log2 = 15
    plans[name] = p


def t(fn):
    fn()
    best = 1e30
    for _ in range(4):
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


res = {}
for name, p in plans.items():
    res[name] = {"map_gather": t(lambda: q.map_gather_planned(p, gates, perm, k1, k2, ws)),
                 "fused": t(lambda: q.run_fused_planned(p, gates, k1, k2, ws))}
    q.build_map(gates, M, perm)
    res[name]["apply"] = t(lambda: q.apply_map_planned(p, perm, k1, k2, ws))
ref = torch.empty_like(perm)
q.build_map(gates, M, ref)
q.map_gather_planned(plans["s6"], gates, perm, k1, k2, ws)
torch.cuda.synchronize()
idx = torch.randint(0, N, (1 << 22,), device=dev)
ok = bool(torch.equal(perm[idx], ref[idx])) and bool(torch.equal(
    k2.view(torch.int64)[idx], k1.view(torch.int64)[ref[idx].long() & 0xffffffff]))
print(json.dumps({"QSIM_STORE_EX": os.environ.get("QSIM_STORE_EX", "1"), "ms": res, "sampled_ok": ok}), flush=True)
