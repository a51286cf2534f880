"""Run one apply variant a few times (for ncu): natural | sigma:<chunk_log2>.

    python tools/profile_apply.py --config cfg5 --variant sigma:12
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--variant", default="natural")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
cfg = wl.CONFIGS[args.config]
gates, M, N = cfg.gates(), cfg.M, cfg.N
e = 8 if cfg.dtype == "c64" else 16
k1 = torch.zeros(N * e, dtype=torch.uint8, device="cuda")
perm = torch.empty(N, dtype=torch.int32, device="cuda")
q.build_map(gates, M, perm)
k2 = torch.empty_like(k1)
if args.variant == "natural":
    fn = lambda: q.apply_map(perm, M, k1, k2, dtype=cfg.dtype)  # noqa: E731
elif args.variant.startswith("sigma"):
    # sigma:<chunk_log2>:<blocks_per_sm>:<dyn>
    f = [int(x) for x in args.variant.split(":")[1:]] + [14, 2, 1][len(args.variant.split(":")) - 1:]
    plan = q.plan_create(gates, M, cfg.dtype)
    plan.chunk_log2, plan.blocks_per_sm = f[0], f[1]
    ws = q.workspace() if f[2] else None
    fn = lambda: q.apply_map_planned(plan, perm, k1, k2, ws)  # noqa: E731
elif args.variant == "fused":
    fn = lambda: q.run_fused(gates, M, k1, k2, dtype=cfg.dtype)  # noqa: E731
elif args.variant.startswith("fsigma"):
    f = [int(x) for x in args.variant.split(":")[1:]] + [14, 2][len(args.variant.split(":")) - 1:]
    plan = q.plan_create(gates, M, cfg.dtype)
    plan.chunk_log2, plan.blocks_per_sm = f[0], f[1]
    ws = q.workspace()
    fn = lambda: q.run_fused_planned(plan, gates, k1, k2, ws)  # noqa: E731
elif args.variant.startswith("mapgather"):
    plan = q.plan_create(gates, M, cfg.dtype)
    ws = q.workspace()
    p2 = torch.empty_like(perm)
    fn = lambda: q.map_gather_planned(plan, gates, p2, k1, k2, ws)  # noqa: E731
elif args.variant == "build":
    fn = lambda: q.build_map(gates, M, perm)  # noqa: E731
for _ in range(args.reps):
    fn()
torch.cuda.synchronize()
print("ok")
