"""Natural vs planned apply / fused on every BASELINE config (cfg2..cfg5).

    python tools/sweep_configs.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402
from tools.sweep_apply import timeit  # noqa: E402


def main():
    for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]:
        cfg = wl.CONFIGS[name]
        gates, M, N = cfg.gates(), cfg.M, cfg.N
        e = 8 if cfg.dtype == "c64" else 16
        k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
        k1.view(torch.int32)[:] = torch.arange(N * e // 4, device="cuda", dtype=torch.int32)
        perm = torch.empty(N, dtype=torch.int32, device="cuda")
        out = torch.empty_like(k1)
        ref = torch.empty_like(k1)
        ws = q.workspace()
        plan = q.plan_create(gates, M, cfg.dtype)
        res = {"config": name, "M": M, "dtype": cfg.dtype}
        res["build_ms"] = timeit(lambda: q.build_map(gates, M, perm))
        res["apply_natural_ms"] = timeit(lambda: q.apply_map(perm, M, k1, ref, dtype=cfg.dtype))
        res["apply_planned_ms"] = timeit(lambda: q.apply_map_planned(plan, perm, k1, out, ws))
        res["apply_equal"] = bool(torch.equal(out, ref))
        res["fused_natural_ms"] = timeit(lambda: q.run_fused(gates, M, k1, out, dtype=cfg.dtype))
        res["fused_planned_ms"] = timeit(lambda: q.run_fused_planned(plan, gates, k1, out, ws))
        res["fused_equal"] = bool(torch.equal(out, ref))
        for k in ("apply_natural", "apply_planned"):
            res[k + "_GBps"] = N * (4 + 2 * e) / res[k + "_ms"] / 1e6
        for k in ("fused_natural", "fused_planned"):
            res[k + "_GBps"] = N * 2 * e / res[k + "_ms"] / 1e6
        res["sigma"] = list(plan.sigma)[:M]
        print(json.dumps(res), flush=True)
        del k1, perm, out, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
