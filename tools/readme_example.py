"""The README's Python example, run as-is (checked on the GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_quant_ph_0308158_b200 as q          # loads libqsim.so (raises if it is missing)

# gates: uint8 rows (kind, target, c0, c1); kind 0 NOT, 1 CNOT, 2 CCNOT, 3 Z, 4 CZ, 5 CCZ, 6 SWAP
gates = np.array([[1, 0, 1, 0], [2, 2, 0, 1], [0, 3, 0, 0]], dtype=np.uint8)
M = 24
k1 = torch.randn(1 << M, dtype=torch.complex64, device="cuda")
k2 = torch.empty_like(k1)
perm = torch.empty(1 << M, dtype=torch.int32, device="cuda")

q.build_map(gates, M, perm)                       # perm[i] = column of row i's unity
q.apply_map(perm, M, k1, k2)                      # k2[i] = k1[perm[i]]
q.run_fused(gates, M, k1, k2)                     # the same k2, map recomputed per entry

plan = q.plan_create(gates, M, "c64")             # traversal order for locality
ws = q.workspace()
q.map_gather_planned(plan, gates, perm, k1, k2, ws)   # perm and k2 in one kernel

qubits = np.tile([0.6, 0.8j], (M, 1))            # row j-1 = [q_j(0), q_j(1)], complex
q.run_fused_kron(gates, M, qubits, k2)            # k1 = q_M (x) ... (x) q_1 generated on the fly
torch.cuda.synchronize()
print("readme example ok")
