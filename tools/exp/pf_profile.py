"""ncu helper: cfg5 fused (or map_gather) with the 13-bit cover plan, each QSIM_PF
variant from argv launched twice (warm-up + measured)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["QSIM_PLAN_COVER_FIXED"] = "1"
import torch
import paper_quant_ph_0308158_b200 as q
import workloads as wl
cfg = wl.CONFIGS["cfg5"]
g, M = cfg.gates(), cfg.M
mode = sys.argv[1]
N = 1 << M
k1 = torch.empty(N * 8, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device="cuda") if mode == "map_gather" else None
ws = q.workspace()
plan = q.plan_create(g, M, "c64")
for v in sys.argv[2:]:
    os.environ["QSIM_PF"] = v
    for _ in range(2):
        if mode == "map_gather":
            q.map_gather_planned(plan, g, perm, k1, k2, ws)
        else:
            q.run_fused_planned(plan, g, k1, k2, ws)
    torch.cuda.synchronize()
    print(v, "done", q.last_kernel(), flush=True)
