"""Sweep scheduling / L2 policy / chunk / occupancy of the sigma gather.

    python tools/sweep_apply2.py --config cfg5
"""
import argparse
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402
from tools.sweep_apply import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--chunks", default="11,12,14,16")
    ap.add_argument("--bps", default="2,4,8")
    ap.add_argument("--ilp", default="16")
    ap.add_argument("--threads", default="256")
    ap.add_argument("--modes", default="apply,fused")
    args = ap.parse_args()
    cfg = wl.CONFIGS[args.config]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    e = 8 if cfg.dtype == "c64" else 16
    k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
    k1.view(torch.int32)[:] = torch.arange(N * e // 4, device="cuda", dtype=torch.int32)
    perm = torch.empty(N, dtype=torch.int32, device="cuda")
    q.build_map(gates, M, perm)
    ref = torch.empty_like(k1)
    q.apply_map(perm, M, k1, ref, dtype=cfg.dtype)
    out = torch.empty_like(k1)
    useful = N * (4 + 2 * e)
    plan = q.plan_create(gates, M, cfg.dtype)
    ws = q.workspace()
    for mode, cl, bps, ilp, thr in itertools.product(args.modes.split(","),
                                                     map(int, args.chunks.split(",")),
                                                     map(int, args.bps.split(",")),
                                                     map(int, args.ilp.split(",")),
                                                     map(int, args.threads.split(","))):
        if cl > M or (ilp == 32 and thr == 1024):
            continue
        plan.chunk_log2, plan.blocks_per_sm, plan.ilp, plan.cta_threads = cl, bps, ilp, thr
        plan.fused_chunk_log2 = cl
        out.zero_()
        if mode == "apply":
            ms = timeit(lambda: q.apply_map_planned(plan, perm, k1, out, ws))
        elif mode == "mapgather":
            pm = torch.empty_like(perm)
            ms = timeit(lambda: q.map_gather_planned(plan, gates, pm, k1, out, ws))
            assert torch.equal(pm, perm)
            del pm
        else:
            ms = timeit(lambda: q.run_fused_planned(plan, gates, k1, out, ws))
        ok = bool(torch.equal(out, ref))
        print(json.dumps({"config": args.config, "mode": mode, "chunk_log2": cl,
                          "bps": bps, "ilp": ilp, "threads": thr, "ms": round(ms, 3), "GBps": round((useful if mode == "apply" else N * 2 * e) / ms / 1e6, 1),
                          "equal": ok}), flush=True)


if __name__ == "__main__":
    main()
