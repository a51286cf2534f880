"""Divergent loads (gather) vs divergent stores (scatter), libqsim_mb.so.

    python tools/mb_scatter.py
"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.sweep_apply import timeit  # noqa: E402

MB = ctypes.CDLL(os.path.join(ROOT, "paper_quant_ph_0308158_b200", "libqsim_mb.so"))
vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32
MB.qsim_mb_gather_c64.argtypes = [vp, u64, vp, vp, i32, i32, i32, vp]
MB.qsim_mb_scatter_c64.argtypes = [vp, u64, vp, vp, i32, i32, vp]


def chk(rc):
    assert rc == 0, rc


def main():
    dev = "cuda"
    st = torch.cuda.current_stream().cuda_stream
    for lr in (22, 26, 28):
        C = 1 << lr
        # a random permutation of [0, C): every output written exactly once
        idx = torch.randperm(C, device=dev).to(torch.int32)
        k1 = torch.empty(C * 8, dtype=torch.uint8, device=dev)
        k1.view(torch.int32)[:] = torch.arange(C * 2, device=dev, dtype=torch.int32)
        out = torch.empty_like(k1)
        for u, b in ((2, 0), (2, 296), (1, 1184)):
            ms = timeit(lambda: chk(MB.qsim_mb_gather_c64(idx.data_ptr(), C, k1.data_ptr(),
                                                         out.data_ptr(), 0, u, b, st)))
            print(json.dumps({"case": f"gather_perm_2^{lr}", "unroll": u, "blocks": b, "ms": ms,
                              "entries_per_s": C / ms * 1e3}), flush=True)
        for u, b in ((8, 0), (16, 296), (4, 1184), (16, 148)):
            ms = timeit(lambda: chk(MB.qsim_mb_scatter_c64(idx.data_ptr(), C, k1.data_ptr(),
                                                          out.data_ptr(), u, b, st)))
            print(json.dumps({"case": f"scatter_perm_2^{lr}", "unroll": u, "blocks": b, "ms": ms,
                              "entries_per_s": C / ms * 1e3}), flush=True)


if __name__ == "__main__":
    main()
