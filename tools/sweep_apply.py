"""Sweep the sigma-ordered gather (qsim_apply_map_planned) on a BASELINE config.

    python tools/sweep_apply.py --config cfg5
Checks every variant's k2 against the natural-order apply (torch.equal).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--chunks", default="8,10,12,14,16,18,20")
    args = ap.parse_args()
    cfg = wl.CONFIGS[args.config]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    e = 8 if cfg.dtype == "c64" else 16
    k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
    k1.view(torch.int32)[:] = torch.arange(N * e // 4, device="cuda", dtype=torch.int32)
    perm = torch.empty(N, dtype=torch.int32, device="cuda")
    q.build_map(gates, M, perm)
    ref = torch.empty_like(k1)
    ms = timeit(lambda: q.apply_map(perm, M, k1, ref, dtype=cfg.dtype))
    useful = N * (4 + 2 * e)
    print(json.dumps({"config": args.config, "variant": "natural k_apply", "ms": ms,
                      "GBps": useful / ms / 1e6}), flush=True)
    plan = q.plan_create(gates, M, cfg.dtype)
    print(json.dumps({"sigma": list(plan.sigma)[:M],
                      "freq": [round(x, 3) for x in list(plan.change_freq)[:M]]}), flush=True)
    out = torch.empty_like(k1)
    for ident in (False, True):
        p2 = q.plan_create(gates, M, cfg.dtype)
        if ident:
            for k in range(32):
                p2.sigma[k] = k
        for cl in map(int, args.chunks.split(",")):
            if cl > M:
                continue
            p2.chunk_log2 = cl
            out.zero_()
            ms = timeit(lambda: q.apply_map_planned(p2, perm, k1, out))
            ok = bool(torch.equal(out, ref))
            print(json.dumps({"config": args.config, "variant": "sigma" if not ident else
                              "identity-sigma", "chunk_log2": cl, "ms": ms,
                              "GBps": useful / ms / 1e6, "equal": ok}), flush=True)


if __name__ == "__main__":
    main()
