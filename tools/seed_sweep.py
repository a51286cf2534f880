"""map+gather time for several random 64-gate circuits at a given M (plan diagnostics).

    python tools/seed_sweep.py --M 32 --seeds 4,5,6,7
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402
from tools.sweep_apply import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=32)
    ap.add_argument("--seeds", default="4,5,6,7")
    ap.add_argument("--ngates", type=int, default=64)
    ap.add_argument("--tune", action="store_true")
    args = ap.parse_args()
    M, N = args.M, 1 << args.M
    k1 = torch.empty(N * 8, dtype=torch.uint8, device="cuda")
    k1.view(torch.int32)[:] = 1
    k2 = torch.empty_like(k1)
    perm = torch.empty(N, dtype=torch.int32, device="cuda")
    ws = q.workspace()
    print("M,seed,map_gather_ms,apply_ms,entries_per_s,spread_nat_log2,spread_sigma_log2,"
          "cover_contained,tuned_variant,sigma")
    for seed in map(int, args.seeds.split(",")):
        gates = wl.random_gates(args.ngates, M, seed)
        plan = q.plan_create(gates, M, "c64")
        variant = -1
        if args.tune:
            variant = q.plan_tune(plan, gates, perm, k1, k2, ws)
        t = timeit(lambda: q.map_gather_planned(plan, gates, perm, k1, k2, ws), reps=3)
        ta = timeit(lambda: q.apply_map_planned(plan, perm, k1, k2, ws), reps=3)
        sp = plan.reserved_spread
        print(f"{M},{seed},{t:.3f},{ta:.3f},{N / t * 1e3:.3e},{sp & 255},{sp >> 8},"
              f"{plan.tile_contained:.3f},{variant},{'-'.join(map(str, list(plan.sigma)[:M]))}", flush=True)


if __name__ == "__main__":
    main()
