"""Many-core driver for the single-threaded oracle -- TEST INFRASTRUCTURE.

The oracle functions stay plain single-threaded C (oracle/qsim_oracle.c); this
module only calls them on disjoint output ranges from host threads (ctypes
releases the GIL), so that the whole 2^32-entry output of BASELINE.json cfg5
can be computed in about a minute and a half on 16 host cores.  The method
shards by output range ("continuous portions"), so the result is the
same bytes as one call over the whole range.  Only tests/ and bench.py's
verification / cpu_baseline legs use it.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _gates_arg, _elem_bytes, _load


def threads_default() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def build_map(gates, M: int, start: int = 0, count: int | None = None,
              threads: int | None = None, out: np.ndarray | None = None,
              piece: int = 1 << 22) -> np.ndarray:
    """perm[start:start+count] (uint32) = oracle_build on pieces of `piece` outputs."""
    if count is None:
        count = (1 << M) - start
    if out is None:
        out = np.empty(count, dtype=np.uint32)
    g, ptr, n = _gates_arg(gates)
    lib = _load()

    def work(a):
        b = min(count, a + piece)
        lib.oracle_build(ptr, n, start + a, b - a, out[a:b].ctypes.data)

    with ThreadPoolExecutor(threads or threads_default()) as ex:
        list(ex.map(work, range(0, count, piece)))
    return out


def apply_map(perm: np.ndarray, k1: np.ndarray, threads: int | None = None,
              out: np.ndarray | None = None, piece: int = 1 << 22) -> np.ndarray:
    """k2[i] = k1[perm[i]] = oracle_apply on pieces of `piece` outputs."""
    count = perm.shape[0]
    if out is None:
        out = np.empty(count, dtype=k1.dtype)
    e = _elem_bytes(k1)
    lib = _load()

    def work(a):
        b = min(count, a + piece)
        lib.oracle_apply(perm[a:b].ctypes.data, b - a, e, k1.ctypes.data, out[a:b].ctypes.data)

    with ThreadPoolExecutor(threads or threads_default()) as ex:
        list(ex.map(work, range(0, count, piece)))
    return out
