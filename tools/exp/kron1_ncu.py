import os, sys
sys.path.insert(0, '/root/repo')
import torch, paper_quant_ph_0308158_b200 as q, workloads as wl
gates = wl.CONFIGS["cfg5"].gates(); qb = wl.random_qubits(32, 2040, "c64")
out = torch.empty(1 << 32, dtype=torch.complex64, device="cuda")
for st in ("1", "0"):
    os.environ["QSIM_KRON_STAGE"] = st
    for i in range(2):
        q.run_fused_kron(gates, 32, qb, out, dtype="c64")
torch.cuda.synchronize()
