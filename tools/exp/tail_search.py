"""Experiment: wider greedy search over the order of the counter bits above
the sector cover (runtime sigma tail), starting from the tuned plan: every
tail bit at every position in [13, 24), best move per round, 4 rounds."""
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
torch.cuda.synchronize()
q.plan_tune(plan, g, perm, k1, k2, ws)
sig = list(plan.sigma)
print("tuned", sig, flush=True)


def t_of(s, reps=3):
    for k in range(32):
        plan.sigma[k] = s[k]
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); q.map_gather_planned(plan, g, perm, k1, k2, ws); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


best = t_of(sig, 5)
print("start", round(best, 3), flush=True)
lo, hi = 13, 24
for rnd in range(4):
    cand = None
    for at in range(lo, M):
        bit = sig[at]
        for pos in range(lo, hi):
            if pos == at:
                continue
            s = sig[:at] + sig[at + 1:]
            s = s[:pos] + [bit] + s[pos:]
            t = t_of(s)
            if cand is None or t < cand[0]:
                cand = (t, s, bit, pos)
    print(f"round {rnd}: best move bit {cand[2]} -> {cand[3]}: {cand[0]:.3f} ms (current {best:.3f})", flush=True)
    if cand[0] < best * 0.995:
        best, sig = cand[0], cand[1]
    else:
        break
print("final", round(t_of(sig, 5), 3), sig, flush=True)
