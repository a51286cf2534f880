import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["QSIM_TUNE_DEBUG"] = "1"
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
torch.cuda.synchronize()
v = q.plan_tune(plan, g, perm, k1, k2, ws)
print("variant", v, list(plan.sigma), plan.chunk_log2, flush=True)
