"""Time qsim_build_map (the materialised map, natural order) for a circuit.
    python tools/bench_build.py M [seed]
(default: cfg5's circuit at M = 32, else random 64 gates seed 4)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

M = int(sys.argv[1])
seed = int(sys.argv[2]) if len(sys.argv) > 2 else None
gates = (wl.random_gates(64, M, seed) if seed is not None
         else wl.CONFIGS["cfg5"].gates() if M == 32 else wl.random_gates(64, M, 4))
N = 1 << M
perm = torch.empty(N, dtype=torch.int32, device="cuda")
times = []
for i in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    q.build_map(gates, M, perm)
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
ms = min(times[2:])
print(f"build M={M} seed={seed}: {ms:.3f} ms {N / ms * 1e3:.3e} entries/s {N * 4 / ms / 1e6:.0f} GB/s "
      f"thread_bits={os.environ.get('QSIM_THREAD_BITS', '-')} [{q.last_kernel()}]")
