"""Multi-process coverage of the N > 1 path on CPU (gloo, world_size 2): sharding covers the
pulse train exactly once, the max-over-ranks time reduction and the result gather."""
import os
import socket

import pytest


def test_shard_range_partitions_exactly():
    from paper_2508_04951_b200.dist import shard_range
    for pulses in (0, 1, 7, 1024, 1023):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                lo, hi = shard_range(pulses, r, world)
                assert 0 <= lo <= hi <= pulses
                got.extend(range(lo, hi))
            assert got == list(range(pulses))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_04951_b200.dist import gather_pulses, max_over_ranks, shard_range
    pulses, n = 5, 16
    lo, hi = shard_range(pulses, rank, world)
    # each rank "processes" its block: marks pulse p with value p (stands in for dc_correct output)
    y = torch.zeros((hi - lo, n), dtype=torch.complex64)
    for i, p in enumerate(range(lo, hi)):
        y[i] = complex(p, -p)
    t = max_over_ranks(10.0 + rank)
    full = gather_pulses(y, pulses)
    q.put((rank, t, full.numpy()))
    dist.destroy_process_group()


def test_gloo_world2_shard_reduce_gather():
    import multiprocessing as mp
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, full in res:
        assert t == 11.0                       # max over ranks
        assert full.shape == (5, 16)
        for p in range(5):
            assert np.all(full[p] == complex(p, -p))
