"""Gather cache-policy / MLP sweep (libqsim_mb.so; not the product path).

    python tools/mb_variants.py [--log2-count 28]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

MB = ctypes.CDLL(os.path.join(ROOT, "paper_quant_ph_0308158_b200", "libqsim_mb.so"))
MB.qsim_mb_gather_c64.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_int32, ctypes.c_void_p]
NAMES = ["nc", "cg", "nc.L1na", "cs", "ca", "L1na", "relaxed.gpu", "nc.L1na.L2_64B"]


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-count", type=int, default=28)
    ap.add_argument("--variants", default="0,1,2,3,4,5,6,7")
    ap.add_argument("--unrolls", default="1,2,4")
    ap.add_argument("--blocks", default="0")
    args = ap.parse_args()
    dev = "cuda"
    N = 1 << 32
    C = 1 << args.log2_count
    k1 = torch.empty(N * 8, dtype=torch.uint8, device=dev)
    k1.view(torch.int64)[:].fill_(7)
    k2 = torch.empty(C * 8, dtype=torch.uint8, device=dev)
    ar = torch.arange(C, device=dev, dtype=torch.int64)
    cases = {"sequential": ar.to(torch.int32)}
    cases["random_2^32"] = torch.randint(0, N, (C,), device=dev, dtype=torch.int64).to(torch.int32)
    for lb in (2, 3):
        blocks = torch.randint(0, N >> lb, (C >> lb,), device=dev, dtype=torch.int64)
        cases[f"block_2^{lb}"] = ((blocks.repeat_interleave(1 << lb) << lb)
                                  | (ar & ((1 << lb) - 1))).to(torch.int32)
    p = torch.empty(C, dtype=torch.int32, device=dev)
    q.build_map_range(wl.CONFIGS["cfg5"].gates(), 32, 0, C, p)
    cases["cfg5"] = p
    st = torch.cuda.current_stream().cuda_stream
    for name, idx in cases.items():
        for v in map(int, args.variants.split(",")):
            for u in map(int, args.unrolls.split(",")):
                for nb in map(int, args.blocks.split(",")):
                    def run():
                        rc = MB.qsim_mb_gather_c64(idx.data_ptr(), C, k1.data_ptr(), k2.data_ptr(),
                                                   v, u, nb, st)
                        assert rc == 0, rc
                    ms = timeit(run)
                    print(json.dumps({"case": name, "variant": NAMES[v], "unroll": u,
                                      "blocks": nb, "ms": round(ms, 4),
                                      "useful_GBps": round(C * 20 / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
