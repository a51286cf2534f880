"""Write-only bandwidth ceiling: torch fill_ / zero_ over a 32 GiB buffer
(the on-the-fly input's output size at M = 32, complex64), CUDA events."""
import torch
N = 1 << 32
out = torch.empty(N, dtype=torch.complex64, device="cuda")
v = out.view(torch.float32)
for name, fn in (("zero_", lambda: v.zero_()), ("fill_", lambda: v.fill_(1.5))):
    ts = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = min(ts[2:])
    print(f"{name}: {ms:.3f} ms  {N * 8 / ms / 1e6:.0f} GB/s written")
