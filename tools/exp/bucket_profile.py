"""ncu helper: cfg3 bucketed fused (and with the map), three calls each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_quant_ph_0308158_b200 as q
import workloads as wl
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = wl.CONFIGS[name]
g, M, N = cfg.gates(), cfg.M, cfg.N
e = 8 if cfg.dtype == "c64" else 16
k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
perm = torch.empty(N, dtype=torch.int32, device="cuda")
for wp in (False, True):
    sc = torch.empty(q.bucket_scratch_bytes(M, cfg.dtype, wp), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        q.run_bucketed(g, M, k1, k2, sc, perm_out=perm if wp else None, dtype=cfg.dtype)
        b.record()
        torch.cuda.synchronize()
        print(name, "with_perm", wp, f"{a.elapsed_time(b):.3f} ms", flush=True)
