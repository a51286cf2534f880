"""Experiment: the cfg5 map + gather step as two independent kernels --
the fused gather (k2 = k1[walk(i)], plan order) and the build (perm in
natural order, coalesced) -- sequential on one stream or concurrent on two,
against the one-pass map+gather kernel (perm stored in plan order).
Results compared byte for byte with the one-pass kernel's."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    cfg = wl.CONFIGS["cfg5"]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    k1 = torch.empty(N * 8, dtype=torch.uint8, device=dev)
    stage = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    chunk = (1 << 30) // 8
    scale = cfg.state.scale()
    for s0 in range(0, N, chunk):
        wl.fill_state(cfg.state, stage.data_ptr(), s0, chunk, scale=scale)
        k1[s0 * 8:(s0 + chunk) * 8].copy_(stage)
    del stage
    k2 = torch.empty_like(k1)
    perm = torch.empty(N, dtype=torch.int32, device=dev)
    ws = q.workspace(dev)
    plan = q.plan_create(gates, M, "c64")
    tuned = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_plan_cfg5.json")))
    for k, v in enumerate(tuned["sigma"]):
        plan.sigma[k] = v
    plan.chunk_log2, plan.fused_chunk_log2 = tuned["chunk_log2"], tuned["fused_chunk_log2"]
    s0 = torch.cuda.current_stream()
    s1 = torch.cuda.Stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    join = torch.cuda.Event()
    fork = torch.cuda.Event()

    def t(fn, reps=6):
        fn()
        torch.cuda.synchronize()
        best = []
        for _ in range(reps):
            ev[0].record(s0)
            fn()
            ev[1].record(s0)
            torch.cuda.synchronize()
            best.append(ev[0].elapsed_time(ev[1]))
        return min(best), sorted(best)[len(best) // 2]

    def one_pass():
        q.map_gather_planned(plan, gates, perm, k1, k2, ws, stream=s0)

    def fused():
        q.run_fused_planned(plan, gates, k1, k2, ws, stream=s0)

    def build():
        q.build_map(gates, M, perm, stream=s0)

    def seq():
        q.run_fused_planned(plan, gates, k1, k2, ws, stream=s0)
        q.build_map(gates, M, perm, stream=s0)

    def par(build_first=False):
        def run():
            fork.record(s0)
            s1.wait_event(fork)
            if build_first:
                q.build_map(gates, M, perm, stream=s1)
                q.run_fused_planned(plan, gates, k1, k2, ws, stream=s0)
            else:
                q.run_fused_planned(plan, gates, k1, k2, ws, stream=s0)
                q.build_map(gates, M, perm, stream=s1)
            join.record(s1)
            s0.wait_event(join)
        return run

    one_pass()
    torch.cuda.synchronize()
    ref_k2 = k2.clone()
    ref_perm = perm.clone()
    res = {}
    for name, fn in (("one_pass map_gather", one_pass), ("fused alone", fused), ("build alone", build),
                     ("fused + build, one stream", seq), ("fused || build, two streams", par()),
                     ("build || fused, two streams (build first)", par(True))):
        k2.zero_()
        perm.zero_()
        r = t(fn)
        ok = None
        if "alone" not in name:
            ok = bool(torch.equal(k2, ref_k2)) and bool(torch.equal(perm, ref_perm))
        res[name] = r
        print(json.dumps({"variant": name, "ms_best": r[0], "ms_med": r[1], "bytes_equal_to_one_pass": ok}),
              flush=True)


if __name__ == "__main__":
    main()
