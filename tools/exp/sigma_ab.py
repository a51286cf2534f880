"""Experiment: A/B of two sigma orders for the cfg5 map+gather, alternating."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_quant_ph_0308158_b200 as q
import workloads as wl
cfg = wl.CONFIGS["cfg5"]
g, M, N = cfg.gates(), cfg.M, cfg.N
k1 = torch.empty(N * 8, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device="cuda")
ws = q.workspace()
plan = q.plan_create(g, M, "c64")
sigs = [json.loads(a) for a in sys.argv[1:]]
base = json.load(open(os.path.join(os.path.dirname(__file__), "..", "..", "profiles", "r02_tuned_plan_cfg5.json")))
plan.chunk_log2 = plan.fused_chunk_log2 = base["chunk_log2"]
plan.flags = base["flags"]
res = {i: [] for i in range(len(sigs))}
for rep in range(8):
    for i, sg in enumerate(sigs):
        for k in range(32):
            plan.sigma[k] = sg[k]
        for r in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); q.map_gather_planned(plan, g, perm, k1, k2, ws); b.record(); torch.cuda.synchronize()
            if rep > 0:
                res[i].append(a.elapsed_time(b))
for i in res:
    v = sorted(res[i])
    print(i, "min", round(v[0], 3), "median", round(v[len(v) // 2], 3), sigs[i][12:22], flush=True)
