"""Experiment (NOT the product path): how the traversal order sigma splits the
cfg5 planned apply's time between its read side and its write side.

first_touch.cu's k_gather takes sigma as a table, so any order can be timed
without JIT: mode 0 = the apply (perm read, k1 gathered, k2 written), mode 5 =
perm read + k2 written (no k1 reads), mode 6 = perm read + k1 gathered (no k2
stores).  Orders: the tuned cfg5 plan, and the tuned plan with output bits
0..k-1 forced onto counter bits 0..k-1 (longer contiguous k2 / perm runs per
warp tile, fewer k1 sector mates inside a CTA)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402
from first_touch import tabs  # noqa: E402


def main():
    reps = int(os.environ.get("OS_REPS", "4"))
    modes = [int(x) for x in os.environ.get("OS_MODES", "0,5,6").split(",")]
    lib = ctypes.CDLL(os.path.join(HERE, "libft.so"))
    dev = torch.device("cuda:0")
    cfg = wl.CONFIGS["cfg5"]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    k1 = torch.empty(N * 2, dtype=torch.float32, device=dev).normal_()
    k2 = torch.empty_like(k1)
    perm = torch.empty(N, dtype=torch.int32, device=dev)
    q.build_map(gates, M, perm)
    tuned = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_plan_cfg5.json")))["sigma"]
    orders = {} if os.environ.get("OS_NO_TUNED") == "1" else {"tuned": tuned}
    for k in [int(x) for x in os.environ.get("OS_FORCE", "5,6,7,8,9,10").split(",") if x]:
        orders[f"low{k}"] = list(range(k)) + [b for b in tuned if b >= k]
    extra = os.environ.get("OS_SIGMA")
    if extra:
        orders["custom"] = [int(x) for x in extra.split(",")]
    bitmap = torch.zeros(N // 32, dtype=torch.int32, device=dev)
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    ticket = torch.zeros(4, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for name, sg in orders.items():
        assert sorted(sg) == list(range(32)), sg
        t = torch.from_numpy(tabs(sg).view(np.int32)).to(dev)
        for chunk_log2 in [int(x) for x in os.environ.get("OS_CHUNK", "15").split(",")]:
            for mode in modes:
                def run():
                    rc = lib.ft_gather(mode, ctypes.c_uint64(N), chunk_log2, ctypes.c_void_p(ticket.data_ptr()),
                                       ctypes.c_void_p(k1.data_ptr()), ctypes.c_void_p(k2.data_ptr()),
                                       ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(bitmap.data_ptr()),
                                       ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(sink.data_ptr()), 148,
                                       ctypes.c_void_p(st))
                    assert rc == 0
                run()
                torch.cuda.synchronize()
                ts = []
                for _ in range(reps):
                    ev[0].record()
                    run()
                    ev[1].record()
                    torch.cuda.synchronize()
                    ts.append(ev[0].elapsed_time(ev[1]))
                print(json.dumps({"order": name, "sigma": sg, "chunk_log2": chunk_log2, "mode": mode,
                                  "ms_best": min(ts), "ms_med": float(np.median(ts))}), flush=True)


if __name__ == "__main__":
    main()
