"""Small invocations of every kernel family for compute-sanitizer (memcheck /
racecheck): natural, planned (sigma and linear), phased, signed build/apply,
input on the fly (32- and 64-bit), ragged ranges.  Exits 0 when all outputs
match the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import oracle  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

dev = "cuda"


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).to(dev)


def main():
    ok = True
    M = 14
    for gates in (wl.random_gates(40, M, 1), wl.random_gates_ext(40, M, 2)):
        k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 3))
        perm_ref, signs_ref = oracle.build_map_signed(gates, M)
        ref = oracle.apply_map_signed(perm_ref, signs_ref, k1)
        k1_d = d(k1)
        for walk in (q.WALK_PER_LANE, q.WALK_BITSLICED):
            out = torch.empty(((1 << M) - 5) * 8, dtype=torch.uint8, device=dev)
            q.run_fused_range(gates, M, 3, (1 << M) - 5, k1_d, out, dtype="c64", walk=walk)
            torch.cuda.synchronize()
            ok &= out.cpu().numpy().tobytes() == ref[3:-2].tobytes()
        plan = q.plan_create(gates, M, "c64")
        plan.flags = 0
        out = torch.empty_like(k1_d)
        q.run_fused_planned(plan, gates, k1_d, out, q.workspace())
        torch.cuda.synchronize()
        ok &= out.cpu().numpy().tobytes() == ref.tobytes()
        perm = torch.empty(1 << M, dtype=torch.int32, device=dev)
        signs = torch.empty((1 << M) // 32, dtype=torch.int32, device=dev)
        q.build_map_signed(gates, M, 0, 1 << M, perm, signs)
        out = torch.empty_like(k1_d)
        q.apply_map_signed(perm, signs, (1 << M) - 1, M, k1_d, out, dtype="c64")
        torch.cuda.synchronize()
        ok &= out.cpu().numpy()[:((1 << M) - 1) * 8].tobytes() == ref[:-1].tobytes()
        if not (gates[:, 0] >= 3).any() or True:
            plain = np.ascontiguousarray(gates[(gates[:, 0] < 3) | (gates[:, 0] == 6)])
            pm = torch.empty(1 << M, dtype=torch.int32, device=dev)
            out = torch.empty_like(k1_d)
            plan2 = q.plan_create(plain, M, "c64")
            plan2.flags = 0
            q.map_gather_planned(plan2, plain, pm, k1_d, out, q.workspace())
            q.build_map_range(plain, M, 7, 1000, perm, walk=q.WALK_JIT)
            torch.cuda.synchronize()
            ok &= np.array_equal(pm.cpu().numpy().view(np.uint32), oracle.build_map(plain, M))
    for MM, cnt in ((12, 4000), (36, 5000)):
        g = wl.random_gates_ext(30, MM, 5)
        qb = wl.random_qubits(MM, 1, "c64")
        for walk in (q.WALK_BITSLICED, q.WALK_JIT, q.WALK_PER_LANE):
            out = torch.empty(cnt, dtype=torch.complex64, device=dev)
            q.run_fused_kron(g, MM, qb, out, start=17, count=cnt, dtype="c64", walk=walk)
            torch.cuda.synchronize()
    print("sanitize cases:", "ok" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
