"""Experiment: per-CTA slice size of the cluster-bucketed pass 2 (QSIM_BUCKET_SLICE_KB)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_quant_ph_0308158_b200 as q
import workloads as wl
cfg = wl.CONFIGS[sys.argv[1]]
g, M, N = cfg.gates(), cfg.M, cfg.N
e = 8 if cfg.dtype == "c64" else 16
k1 = torch.empty(N * e, dtype=torch.uint8, device="cuda")
torch.arange(k1.numel() // 8, out=k1.view(torch.int64))
k2 = torch.empty_like(k1)
ref = None
for kb in sys.argv[2:]:
    os.environ["QSIM_BUCKET_SLICE_KB"] = kb
    nb = q.bucket_scratch_bytes(M, cfg.dtype, False)
    if nb == 0:
        print(kb, "out of range"); continue
    sc = torch.empty(nb, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); q.run_bucketed(g, M, k1, k2, sc, dtype=cfg.dtype); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    if ref is None:
        ref = k2.clone()
    print(f"slice {kb} KB: {min(ts[1:]):.3f} ms  equal {bool(torch.equal(k2, ref))}", flush=True)
    del sc
