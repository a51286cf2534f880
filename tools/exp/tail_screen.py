"""Experiment: replicate qsim_plan_tune's stage-3 screening from a given sigma
(one timed call per move) and print the best moves."""
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
plan.chunk_log2 = plan.fused_chunk_log2 = 15
plan.flags = 0
cur = json.loads(sys.argv[1])
def t_of(s, reps):
    for k in range(32):
        plan.sigma[k] = s[k]
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); q.map_gather_planned(plan, g, perm, k1, k2, ws); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)
t_of(cur, 2)
print("cur", t_of(cur, 3))
res = []
frm = int(sys.argv[2]) if len(sys.argv) > 2 else 13
for at in range(frm, M):
    for pos in range(frm, frm + 10):
        if pos == at:
            continue
        s = cur[:at] + cur[at + 1:]
        s = s[:pos] + [cur[at]] + s[pos:]
        res.append((t_of(s, 1), cur[at], pos))
res.sort()
for r in res[:10]:
    print(r)
