"""Host-only: how well can an aligned block of 2^T outputs (a CTA or a
thread-block cluster) contain the readers of one 128-byte k1 line?

For sampled k1 lines L (16 complex64 entries) the 16 readers are
g(16 L + r) (g = perm^-1, Step 1 first).  For T = 13..20 a greedy cover
picks T output bits (starting from the kept bits 0..2, adding the commonest
reader-difference patterns, as qsim_plan's sector cover does for 32-byte
sectors) and reports
  * pairs: fraction of (reader, line-mate reader) pairs inside one block,
  * blocks_per_line: mean number of distinct blocks a line's readers fall in
    (= k1 line fetches per line if each block fetched its lines whole),
  * whole: fraction of lines whose 16 readers all fall in one block.
A block-staged design (each CTA / cluster fetches its blocks' k1 lines whole
and serves the readers from shared / distributed shared memory) moves
blocks_per_line x the k1 bytes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as wl  # noqa: E402


def fwd(gates, x):
    x = x.copy()
    one = np.uint64(1)
    for k, t, c0, c1 in gates:
        t = np.uint64(t)
        if k == 0:
            x ^= one << t
        elif k == 1:
            x ^= ((x >> np.uint64(c0)) & one) << t
        else:
            x ^= (((x >> np.uint64(c0)) & (x >> np.uint64(c1))) & one) << t
    return x


def main(name="cfg5", lines=4096, lb=4):
    cfg = wl.CONFIGS[name]
    g, M = cfg.gates(), cfg.M
    rng = np.random.default_rng(7)
    L = rng.integers(0, 1 << (M - lb), lines, dtype=np.uint64)
    src = (L[:, None] << np.uint64(lb)) | np.arange(1 << lb, dtype=np.uint64)[None, :]
    rd = fwd(g, src.ravel()).reshape(src.shape)
    d = (rd[:, 1:] ^ rd[:, :1]).ravel()           # differences to the first reader
    pats, cnt = np.unique(d, return_counts=True)
    order = np.argsort(-cnt)[:512]
    pats, cnt = pats[order], cnt[order]
    full = (1 << M) - 1
    print(f"# {name}: M={M}, {lines} sampled k1 lines of {1 << lb} entries; greedy cover over the "
          f"512 commonest reader-difference patterns")
    print("T  pairs  blocks_per_line  whole")
    for T in range(13, 21):
        V = 7
        while bin(V).count("1") < T:
            best, add = -1.0, 0
            for p in pats:
                a = int(p) & ~V
                na = bin(a).count("1")
                if na == 0 or bin(V).count("1") + na > T:
                    continue
                gain = cnt[(pats & np.uint64(full & ~(V | a))) == 0].sum() / na
                if gain > best:
                    best, add = gain, a
            if add == 0:
                add = next(1 << b for b in range(M) if not (V >> b) & 1)
            V |= add
        hi = rd & np.uint64(full & ~V)
        pairs = float(((d & np.uint64(full & ~V)) == 0).mean())
        srt = np.sort(hi, axis=1)
        nb = 1 + (srt[:, 1:] != srt[:, :-1]).sum(axis=1)
        print(f"{T:2d} {pairs:6.3f} {nb.mean():8.2f} {float((nb == 1).mean()):8.3f}")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["cfg5"]))
