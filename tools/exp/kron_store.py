"""Experiment: store policy of the on-the-fly input kernel (QSIM_KRON_ST)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_quant_ph_0308158_b200 as q
import workloads as wl
N = 1 << 32
k2 = torch.empty(N * 8, dtype=torch.uint8, device="cuda")
cases = [(32, wl.CONFIGS["cfg5"].gates(), 0), (40, wl.random_gates(64, 40, 4), (1 << 39) - (1 << 31))]
ref = {}
for st in sys.argv[1:]:
    os.environ["QSIM_KRON_ST"] = st
    for M, g, start in cases:
        qb = wl.random_qubits(M, 2024, "c64")
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); q.run_fused_kron(g, M, qb, k2, start=start, count=N, dtype="c64"); b.record()
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        h = int(k2.view(torch.int64)[::4097].sum().item())
        ok = ref.setdefault(M, h) == h
        print(f"st={st} M={M}: {min(ts[1:]):.3f} ms  same {ok}", flush=True)
