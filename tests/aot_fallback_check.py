"""Run under QSIM_NO_JIT=1 (the ahead-of-time kernels only): planned apply /
fused / map+gather over every launch shape of the AOT sigma kernels (CTA
threads 256/512/1024 x gathers in flight 8/16/32, except 32 x 1024), complex64 and complex128,
byte for byte against the oracle.  Invoked by tests/test_gpu_parity.py in a
subprocess (the JIT switch is read once per process)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
assert os.environ.get("QSIM_NO_JIT") == "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

assert not q.jit_status().startswith("ready"), q.jit_status()
M = 16
gates = wl.random_gates(64, M, 31)
perm_ref = oracle.build_map(gates, M)
ws = q.workspace()
for dtype in ("c64", "c128"):
    k1 = wl.make_state(wl.StateSpec(M, dtype, wl.GAUSS, 5))
    ref = oracle.apply_map(perm_ref, k1).tobytes()
    k1_d = torch.from_numpy(k1.view(np.uint8)).cuda()
    perm_d = torch.from_numpy(perm_ref.view(np.int32)).cuda()
    for threads in (256, 512, 1024):
        for ilp in (8, 16, 32):
            if ilp == 32 and threads == 1024:
                continue              # rejected by qsim_plan validation (register file)
            plan = q.plan_create(gates, M, dtype)
            plan.flags &= ~1          # the plan's order, not natural
            plan.cta_threads = threads
            plan.ilp = ilp
            for call in ("apply", "fused", "map_gather"):
                k2_d = torch.zeros_like(k1_d)
                pm = torch.zeros_like(perm_d)
                if call == "apply":
                    q.apply_map_planned(plan, perm_d, k1_d, k2_d, ws)
                elif call == "fused":
                    q.run_fused_planned(plan, gates, k1_d, k2_d, ws)
                else:
                    q.map_gather_planned(plan, gates, pm, k1_d, k2_d, ws)
                torch.cuda.synchronize()
                assert k2_d.cpu().numpy().tobytes() == ref, (dtype, threads, ilp, call, q.last_kernel())
                if call == "map_gather":
                    assert np.array_equal(pm.cpu().numpy().view(np.uint32), perm_ref)
# input on the fly without NVRTC (identity table layout), within the rounding bound
import math  # noqa: E402
Mk = 22
gk = wl.random_gates(64, Mk, 8)
for dtype in ("c64", "c128"):
    qb = wl.random_qubits(Mk, 4, dtype)
    out = torch.empty(1 << Mk, dtype=torch.complex64 if dtype == "c64" else torch.complex128, device="cuda")
    q.run_fused_kron(gk, Mk, qb, out, dtype=dtype)
    torch.cuda.synchronize()
    assert q.last_kernel() == "k_fused_kron_bitsliced", q.last_kernel()
    ref = oracle.fused_kron(gk, qb)
    u = 2.0 ** -24 if dtype == "c64" else 2.0 ** -53
    err = np.abs(out.cpu().numpy().astype(np.complex128) - ref)
    assert np.all(err <= 1.01 * (Mk - 1) * math.sqrt(5.0) * u * np.abs(ref)), dtype
print("aot fallback ok")
