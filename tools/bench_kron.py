"""Time qsim_run_fused_kron (input on the fly) for a circuit and a portion.
    python tools/bench_kron.py M [count_log2] [dtype] [seed]
(seed: random 64-gate circuit; default cfg5's circuit at M = 32, seed 4 otherwise)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

M = int(sys.argv[1])
cl = int(sys.argv[2]) if len(sys.argv) > 2 else min(M, 32)
dtype = sys.argv[3] if len(sys.argv) > 3 else "c64"
seed = int(sys.argv[4]) if len(sys.argv) > 4 else None
gates = (wl.random_gates(64, M, seed) if seed is not None
         else wl.CONFIGS["cfg5"].gates() if M == 32 else wl.random_gates(64, M, 4))
qb = wl.random_qubits(M, 2040, dtype)
count = 1 << cl
start = 0 if count == (1 << M) else (1 << (M - 1)) - count // 2
out = torch.empty(count, dtype=torch.complex64 if dtype == "c64" else torch.complex128, device="cuda")
times = []
for i in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    q.run_fused_kron(gates, M, qb, out, start=start, count=count, dtype=dtype)
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
ms = min(times[2:])
e = 8 if dtype == "c64" else 16
print(f"M={M} count=2^{cl} {dtype} {ms:.3f} ms "
      f"{count / ms * 1e3:.3e} entries/s {count * e / ms / 1e6:.0f} GB/s seed={seed} "
      f"layout={os.environ.get('QSIM_THREAD_BITS', '-')} [{q.last_kernel()}]")
