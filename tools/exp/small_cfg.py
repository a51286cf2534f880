"""Experiment: where the launch-bound cfg2 step (M = 20, L2-resident) spends
its time.  Times qsim_map_gather_planned / run_fused_planned with and without
the workspace ticket, direct and from a CUDA graph, warm."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.Stream(dev)
for name in os.environ.get("CFGS", "cfg2").split(","):
    c = wl.CONFIGS[name]
    g, N, M = c.gates(), c.N, c.M
    e = 8 if c.dtype == "c64" else 16
    a = torch.randn(N, dtype=torch.complex64 if e == 8 else torch.complex128, device=dev)
    b = torch.empty_like(a)
    p = torch.empty(N, dtype=torch.int32, device=dev)
    plan = q.plan_create(g, M, c.dtype)
    ws = q.workspace(dev)
    reps = int(os.environ.get("REPS", "200"))
    for call, fn in (("map_gather ws", lambda: q.map_gather_planned(plan, g, p, a, b, ws, stream=st)),
                     ("map_gather no-ws", lambda: q.map_gather_planned(plan, g, p, a, b, None, stream=st)),
                     ("fused ws", lambda: q.run_fused_planned(plan, g, a, b, ws, stream=st)),
                     ("fused no-ws", lambda: q.run_fused_planned(plan, g, a, b, None, stream=st)),
                     ("plain run_fused", lambda: q.run_fused(g, M, a, b, stream=st)),
                     ("build_map", lambda: q.build_map(g, M, p, stream=st))):
        with torch.cuda.stream(st):
            fn()
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2000000)
            t0.record(st)
            for _ in range(reps):
                fn()
            t1.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"cfg": name, "call": call, "us_per_call": 1e3 * t0.elapsed_time(t1) / reps,
                          "kernel": q.last_kernel(), "flags": plan.flags,
                          "chunk_log2": plan.fused_chunk_log2}), flush=True)
