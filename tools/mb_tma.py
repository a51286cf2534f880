"""TMA tile::gather4 vs LSU gather microbenchmark (libqsim_mb.so).

    python tools/mb_tma.py
"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402
from tools.sweep_apply import timeit  # noqa: E402

MB = ctypes.CDLL(os.path.join(ROOT, "paper_quant_ph_0308158_b200", "libqsim_mb.so"))
vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32
MB.qsim_mb_gather_c64.argtypes = [vp, u64, vp, vp, i32, i32, i32, vp]
MB.qsim_mb_tma_gather_c64.argtypes = [vp, u64, vp, u64, vp, i32, i32, vp]


def chk(rc):
    assert rc == 0, rc


def main():
    N = 1 << 32
    C = 1 << 28
    dev = "cuda"
    k1 = torch.empty(N * 8, dtype=torch.uint8, device=dev)
    k1.view(torch.int32)[:] = torch.arange(N * 2, device=dev, dtype=torch.int32)
    ref = torch.empty(C * 8, dtype=torch.uint8, device=dev)
    out = torch.empty_like(ref)
    st = torch.cuda.current_stream().cuda_stream
    cases = {}
    cases["sequential"] = torch.arange(C, device=dev, dtype=torch.int64).to(torch.int32)
    cases["random_region_2^22"] = torch.randint(0, 1 << 22, (C,), device=dev).to(torch.int32)
    cases.pop("sequential")
    cases["random_2^32"] = torch.randint(0, N, (C,), device=dev, dtype=torch.int64).to(torch.int32)
    # the cfg5 source stream in sigma order (first 2^28 counters)
    cfg = wl.CONFIGS["cfg5"]
    gates = cfg.gates()
    plan = q.plan_create(gates, 32, "c64")
    perm = torch.empty(N, dtype=torch.int32, device=dev)
    q.build_map(gates, 32, perm)
    c = torch.arange(C, device=dev, dtype=torch.int64)
    out_idx = torch.zeros(C, device=dev, dtype=torch.int64)
    for k in range(32):
        out_idx |= ((c >> k) & 1) << int(plan.sigma[k])
    cases["cfg5_sigma_stream"] = perm[out_idx]
    del out_idx, c, perm
    useful = C * 20
    for name, idx in cases.items():
        ms = timeit(lambda: chk(MB.qsim_mb_gather_c64(idx.data_ptr(), C, k1.data_ptr(),
                                                     ref.data_ptr(), 0, 2, 0, st)))
        print(json.dumps({"case": name, "impl": "ldg", "ms": round(ms, 3),
                          "useful_GBps": round(useful / ms / 1e6, 1)}), flush=True)
        for stages, blocks in ((404, 296), (802, 296), (803, 148), (1602, 148), (1601, 296),
                               (1202, 148), (802, 444)):
                out.zero_()
                ms = timeit(lambda: chk(MB.qsim_mb_tma_gather_c64(idx.data_ptr(), C, k1.data_ptr(), N,
                                                                 out.data_ptr(), stages, blocks,
                                                                 st)))
                ok = bool(torch.equal(out, ref))
                print(json.dumps({"case": name, "impl": "tma_gather4", "stages": stages % 100, "producers": stages // 100,
                                  "blocks": blocks, "ms": round(ms, 3),
                                  "useful_GBps": round(useful / ms / 1e6, 1), "equal": ok}),
                      flush=True)


if __name__ == "__main__":
    main()
