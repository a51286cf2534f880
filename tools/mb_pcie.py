"""PCIe copy rates on the B200 host link (pinned buffers): H2D alone, D2H alone,
both at once on two streams, and chunked variants.  Prints JSON lines."""
import json
import time

import torch

GB = 1 << 30
n = 8 * GB
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


def both_chunked(c=256 << 20):
    for o in range(0, n, c):
        with torch.cuda.stream(s1):
            d1[o:o + c].copy_(h1[o:o + c], non_blocking=True)
        with torch.cuda.stream(s2):
            h2[o:o + c].copy_(d2[o:o + c], non_blocking=True)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("both_chunked_256MB", both_chunked)):
    t = run(fn)
    print(json.dumps({"case": name, "s": round(t, 4), "GBps_each_direction": n / t / 1e9}), flush=True)


# round 2: more streams per direction, other chunk sizes
s3, s4 = torch.cuda.Stream(), torch.cuda.Stream()


def both_4streams(c=256 << 20):
    for i, o in enumerate(range(0, n, c)):
        with torch.cuda.stream(s1 if i % 2 == 0 else s3):
            d1[o:o + c].copy_(h1[o:o + c], non_blocking=True)
        with torch.cuda.stream(s2 if i % 2 == 0 else s4):
            h2[o:o + c].copy_(d2[o:o + c], non_blocking=True)


for name, fn in (("both_chunked_64MB", lambda: both_chunked(64 << 20)),
                 ("both_chunked_1GB", lambda: both_chunked(1 << 30)),
                 ("both_4streams_256MB", both_4streams),
                 ("both_4streams_64MB", lambda: both_4streams(64 << 20))):
    t = run(fn)
    print(json.dumps({"case": name, "s": round(t, 4), "GBps_each_direction": n / t / 1e9}), flush=True)
