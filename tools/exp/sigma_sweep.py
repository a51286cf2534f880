"""Experiment: reorder the non-cover part of the tuned plan's sigma so that
output bits next to the k2 / perm store runs (write-side DRAM row locality)
sit at lower counter bits.  Variant: comma list of output bits moved to just
after the cover, in that order ("-" = tuned plan as is)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_quant_ph_0308158_b200 as q
import workloads as wl

cfg = wl.CONFIGS["cfg5"]
g, M = cfg.gates(), cfg.M
N = 1 << M
k1 = torch.empty(N * 8, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device="cuda")
ws = q.workspace()
plan = q.plan_create(g, M, "c64")
torch.cuda.synchronize()
q.plan_tune(plan, g, perm, k1, k2, ws)
base = list(plan.sigma)
T = plan.tile_log2
print("tuned", base, "cover", T, flush=True)
q.map_gather_planned(plan, g, perm, k1, k2, ws)
torch.cuda.synchronize()
k2_ref, perm_ref = k2.clone(), perm.clone()

def timeit(fn, reps=4):
    ts = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])

for v in sys.argv[1:]:
    sig = list(base)
    if v != "-":
        pos, bits = v.split(":") if ":" in v else (str(13), v)
        pos = int(pos)
        mv = [int(b) for b in bits.split(",")]
        rest = [b for b in sig[pos:] if b not in mv]
        sig = sig[:pos] + mv + rest
        assert sorted(sig) == list(range(32)), sig
    for k in range(32):
        plan.sigma[k] = sig[k]
    k2.zero_()
    mg = timeit(lambda: q.map_gather_planned(plan, g, perm, k1, k2, ws))
    ok = bool(torch.equal(k2, k2_ref)) and bool(torch.equal(perm, perm_ref))
    fu = timeit(lambda: q.run_fused_planned(plan, g, k1, k2, ws))
    ok = ok and bool(torch.equal(k2, k2_ref))
    print(f"{v:24s} mg {mg:.3f} fu {fu:.3f} {'ok' if ok else 'MISMATCH'} sigma {sig}", flush=True)
