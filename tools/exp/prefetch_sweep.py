"""Experiment: granule prefetch ahead of the gather (QSIM_PF="mode,D,G"), cfg5.
Variant syntax: "mode,D,G[,W[,chunk_log2]]".  Prints per variant the steady-state
times of the selected calls (mg = map+gather, fu = fused, ap = apply) and
whether the outputs equal the no-prefetch run byte for byte."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_quant_ph_0308158_b200 as q
import workloads as wl

cfg = wl.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
variants = sys.argv[2].split(";") if len(sys.argv) > 2 else ["0,0,4"]
calls = sys.argv[3].split(",") if len(sys.argv) > 3 else ["mg", "fu"]
g, M = cfg.gates(), cfg.M
e = 8 if cfg.dtype == "c64" else 16
N = 1 << M
k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device="cuda")
ws = q.workspace()
os.environ.pop("QSIM_PF", None)
plan = q.plan_create(g, M, cfg.dtype)
torch.cuda.synchronize()
tuned = q.plan_tune(plan, g, perm, k1, k2, ws)
print("tuned variant", tuned, list(plan.sigma), plan.fused_chunk_log2, flush=True)
c0 = plan.fused_chunk_log2

def timeit(fn, reps=5):
    ts = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:]), sorted(ts[1:])[len(ts[1:]) // 2]

q.map_gather_planned(plan, g, perm, k1, k2, ws)
torch.cuda.synchronize()
k2_ref, perm_ref = k2.clone(), perm.clone()
run = {"mg": lambda: q.map_gather_planned(plan, g, perm, k1, k2, ws),
       "fu": lambda: q.run_fused_planned(plan, g, k1, k2, ws),
       "ap": lambda: q.apply_map_planned(plan, perm_ref, k1, k2, ws)}
for v in variants:
    parts = v.split(",")
    os.environ["QSIM_PF"] = ",".join(parts[:4])
    plan.chunk_log2 = plan.fused_chunk_log2 = int(parts[4]) if len(parts) > 4 else c0
    out = []
    for c in calls:
        k2.zero_()
        t = timeit(run[c])
        ok = bool(torch.equal(k2, k2_ref)) and (c != "mg" or bool(torch.equal(perm, perm_ref)))
        out.append(f"{c} min {t[0]:.3f} med {t[1]:.3f} {'ok' if ok else 'MISMATCH'} {q.last_kernel()}")
    print(f"PF={v:12s} " + " | ".join(out) + f"  [{q.last_kernel()}]", flush=True)
