"""The bench's step kernels one at a time, for ncu.

    python tools/profile_step.py tune  plan.json     # plan_create + plan_tune (no ncu), save the plan
    python tools/profile_step.py run   plan.json CALL [reps]
        CALL: map_gather | fused | apply | build | kron | plain_fused
Each run call launches the kernel `reps` times (default 2: a warm-up and one
to capture with `ncu -s 1 -c 1`)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
cfg = wl.CONFIGS[os.environ.get("QSIM_PROFILE_CONFIG", "cfg5")]
g, M, N = cfg.gates(), cfg.M, cfg.N
e = 8 if cfg.dtype == "c64" else 16
k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device="cuda")
ws = q.workspace()
plan = q.plan_create(g, M, cfg.dtype)
if mode == "tune":
    torch.cuda.synchronize()
    v = q.plan_tune(plan, g, perm, k1, k2, ws)
    with open(path, "w") as f:
        json.dump({"variant": v, "sigma": list(plan.sigma), "chunk_log2": plan.chunk_log2,
                   "fused_chunk_log2": plan.fused_chunk_log2, "blocks_per_sm": plan.blocks_per_sm,
                   "flags": plan.flags}, f)
    print("tuned", v, list(plan.sigma))
    sys.exit(0)
with open(path) as f:
    saved = json.load(f)
for k, b in enumerate(saved["sigma"]):
    plan.sigma[k] = b
plan.chunk_log2, plan.fused_chunk_log2 = saved["chunk_log2"], saved["fused_chunk_log2"]
plan.blocks_per_sm, plan.flags = saved["blocks_per_sm"], saved["flags"]
call = sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
if call == "apply":
    q.build_map(g, M, perm)
qb = wl.random_qubits(M, 2024, cfg.dtype)
fn = {"map_gather": lambda: q.map_gather_planned(plan, g, perm, k1, k2, ws),
      "fused": lambda: q.run_fused_planned(plan, g, k1, k2, ws),
      "apply": lambda: q.apply_map_planned(plan, perm, k1, k2, ws),
      "build": lambda: q.build_map(g, M, perm),
      "kron": lambda: q.run_fused_kron(g, M, qb, k2, dtype=cfg.dtype),
      "plain_fused": lambda: q.run_fused(g, M, k1, k2, dtype=cfg.dtype)}[call]
for _ in range(reps):
    fn()
torch.cuda.synchronize()
print(call, "done", q.last_kernel())
