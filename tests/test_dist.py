"""Multi-process host logic on CPU (gloo, world_size 2): output-range
sharding (the paper's "continuous portions") and the bench's
max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest

from paper_quant_ph_0308158_b200.dist import output_shards


@pytest.mark.parametrize("N,world", [(8, 1), (8, 2), (1 << 20, 2), (1 << 20, 3), (5000, 4),
                                     (1 << 32, 8), (3, 8)])
def test_output_shards_cover_exactly_once(N, world):
    sh = output_shards(N, world)
    assert len(sh) == world
    pos = 0
    for start, count in sh:
        assert start == pos and count >= 0
        pos += count
    assert pos == N
    for start, _ in sh[1:]:
        assert start % 1024 == 0 or start == N


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    import workloads as wl
    from paper_quant_ph_0308158_b200.dist import barrier, max_over_ranks, output_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M = 14
        gates = wl.random_gates(64, M, 5)
        k1 = wl.make_state(wl.StateSpec(M, "c64", wl.GAUSS, 5))      # replicated input
        start, count = output_shards(1 << M, world)[rank]
        mine = oracle.run_fused(gates, k1, start, count)            # this rank's portion
        parts = [None] * world
        dist.all_gather_object(parts, (start, mine.tobytes()))
        barrier()
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            glued = b"".join(p for _, p in sorted(parts))
            full = oracle.apply_map(oracle.build_map(gates, M), k1).tobytes()
            q.put((glued == full, t))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_path():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    equal, tmax = q.get(timeout=10)
    assert equal
    assert tmax == 2.0
