"""Time the planned calls call by call (the first call includes NVRTC compile).

    python tools/diag_planned.py CFG MODE [key=value ...]
      CFG   cfg1..cfg5, rand:M (64 random gates over M bits, seed 4), seed:S (M = 32,
            64 random gates, seed S), low:B / high:B
            (M = 32, 64 random gates on bits < B / >= B)
      MODE  fused | map_gather | apply
      keys  order=plan|natural|sigma (sigma forces the plan's order),
            chunk=<log2>, bps=<blocks per SM>, T=<cover bits, informational>
Prints one line per call; the last is the steady-state time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

name, mode = sys.argv[1], sys.argv[2]
kv = dict(a.split("=") for a in sys.argv[3:])
if name.startswith("rand:"):
    M = int(name[5:])
    g, dtype = wl.random_gates(64, M, 4), "c64"
elif name.startswith("seed:"):
    M, dtype = 32, "c64"
    g = wl.random_gates(64, 32, int(name[5:]))
elif name.startswith("low:") or name.startswith("high:"):
    # M=32 circuits that keep locality: every gate on bits < B (low:B) or >= B (high:B)
    kind, B = name.split(":")
    M, dtype = 32, "c64"
    bits = list(range(int(B))) if kind == "low" else list(range(int(B), 32))
    import numpy as np
    rng = np.random.default_rng(11)
    rows = []
    for _ in range(64):
        k = int(rng.integers(3))
        b = rng.choice(bits, size=1 + k, replace=False)
        rows.append(wl.gate(k, int(b[0]), *[int(x) for x in b[1:]]))
    g = wl.gates_array(rows)
else:
    cfg = wl.CONFIGS[name]
    g, M, dtype = cfg.gates(), cfg.M, cfg.dtype
e = 8 if dtype == "c64" else 16
N = 1 << M
k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device="cuda")
ws = q.workspace()
plan = q.plan_create(g, M, dtype)
order = kv.get("order", "plan")
if order == "natural":
    plan.flags |= 1
elif order == "sigma":
    plan.flags &= ~1
if "chunk" in kv:
    plan.chunk_log2 = plan.fused_chunk_log2 = int(kv["chunk"])
if "bps" in kv:
    plan.blocks_per_sm = int(kv["bps"])
q.build_map(g, M, perm)
run = {"fused": lambda: q.run_fused_planned(plan, g, k1, k2, ws),
       "map_gather": lambda: q.map_gather_planned(plan, g, perm, k1, k2, ws),
       "apply": lambda: q.apply_map_planned(plan, perm, k1, k2, ws)}[mode]
for i in range(4):
    t = time.time()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"{name} {mode} {' '.join(sys.argv[3:])} call {i}: {ms:.3f} ms  entries/s {N / ms * 1e3:.3e}"
          f"  launches {q.lib().qsim_last_launch_count()}  natural {plan.flags & 1}"
          f"  chunk {plan.chunk_log2}  contained {plan.tile_contained:.3f}"
          f"  [{q.last_kernel()}]", flush=True)
