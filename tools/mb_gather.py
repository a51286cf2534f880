"""Gather microbenchmarks on B200 (not part of the product path).

Times the product gather kernel (qsim_apply_map_range, complex64) on index
streams with controlled locality, to locate the ceiling of the apply step:
sequential, random within a region of R entries (TLB reach / L2 residency),
block-shuffled with block size B (DRAM granule), random within 2 MB pages
visited in order, and the cfg5 map itself.  Prints one JSON line per case.

    python tools/mb_gather.py [--log2-count 28]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402


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
    ap.add_argument("--log2-k1", type=int, default=32)
    args = ap.parse_args()
    dev = "cuda"
    Mk = args.log2_k1
    N = 1 << Mk
    C = 1 << args.log2_count
    k1 = torch.empty(N * 8, dtype=torch.uint8, device=dev)
    k1.view(torch.int64)[:].fill_(7)
    k2 = torch.empty(C * 8, dtype=torch.uint8, device=dev)

    def report(name, idx, extra=None):
        ms = timeit(lambda: q.apply_map_range(idx, C, Mk, k1, k2, dtype="c64"))
        useful = C * 20
        line = {"case": name, "ms": ms, "useful_GBps": useful / ms / 1e6,
                "entries_per_s": C / ms * 1e3}
        if extra:
            line.update(extra)
        print(json.dumps(line), flush=True)

    # torch copy reference (read + write), 2 x 8 GiB
    src = k1[: 1 << 33]
    dst = torch.empty_like(src)
    ms = timeit(lambda: dst.copy_(src))
    print(json.dumps({"case": "torch_copy_8GiB", "ms": ms, "GBps": 2 * src.numel() / ms / 1e6}),
          flush=True)
    del dst, src

    ar = torch.arange(C, device=dev, dtype=torch.int64)
    report("sequential", ar.to(torch.int32))
    for lr in (14, 16, 18, 20, 22, 24, 26, 28, 30, 32):
        if lr > Mk:
            continue
        idx = torch.randint(0, 1 << lr, (C,), device=dev, dtype=torch.int64).to(torch.int32)
        report(f"random_region_2^{lr}", idx, {"region_MiB": (8 << lr) >> 20})
        del idx
    for lb in (2, 3, 4, 5, 8, 12, 18):
        nb = C >> lb
        blocks = torch.randint(0, N >> lb, (nb,), device=dev, dtype=torch.int64)
        idx = ((blocks.repeat_interleave(1 << lb) << lb) | (ar & ((1 << lb) - 1))).to(torch.int32)
        report(f"block_random_B=2^{lb}", idx, {"block_bytes": 8 << lb})
        del idx, blocks
    # random within 2 MB pages, pages in order
    idx = ((ar >> 18) << 18) | torch.randint(0, 1 << 18, (C,), device=dev, dtype=torch.int64)
    report("random_within_2MB_pages_in_order", idx.to(torch.int32))
    idx = ((ar >> 15) << 15) | torch.randint(0, 1 << 15, (C,), device=dev, dtype=torch.int64)
    report("random_within_256KB_in_order", idx.to(torch.int32))
    del idx
    # the cfg5 map (first C outputs of the real perm)
    if Mk == 32:
        gates = wl.CONFIGS["cfg5"].gates()
        p = torch.empty(C, dtype=torch.int32, device=dev)
        q.build_map_range(gates, 32, 0, C, p)
        report("cfg5_perm_first_outputs", p)
        gates4 = wl.CONFIGS["cfg4"].gates()
        q.build_map_range(gates4, 30, 0, C, p)
        report("cfg4_perm_first_outputs(k1 2^32 buffer)", p)


if __name__ == "__main__":
    main()
