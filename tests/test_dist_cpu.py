"""Multi-rank host logic on CPU (gloo, world_size 2): segment sharding, local
views, and the exact byte allgather the library's collectives run on."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2401_00109_b200 import api


@pytest.mark.parametrize("steps,world", [([100] * 10, 2), ([5, 500, 5, 5, 5, 5, 500], 3),
                                         ([1, 1], 2), ([99999] * 10000, 8)])
def test_shard_segments_partition(steps, world):
    cover = []
    loads = []
    for r in range(world):
        s0, s1 = api.shard_segments(steps, world, r)
        assert s1 > s0
        cover += list(range(s0, s1))
        loads.append(sum(steps[s0:s1]))
    assert cover == list(range(len(steps)))
    if len(set(steps)) == 1:
        assert max(loads) - min(loads) <= steps[0]


def test_local_view_split_series_shares_boundaries():
    first, steps = api.plan_segments([1001], 0, 8)
    x = np.arange(1001.0)
    got = []
    for r in range(3):
        s0, s1 = api.shard_segments(steps, 3, r)
        lo, hi, lf, ls = api.local_view(first, steps, s0, s1)
        v = x[lo:hi + 1]
        for f, s in zip(lf, ls):
            got.append((v[f], v[f + s]))
    assert got == [(x[f], x[f + s]) for f, s in zip(first, steps)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import ctypes as C

    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    comm = api.TorchComm()
    payload = np.arange(5, dtype=np.int64) * (rank + 1)
    recv = np.zeros(5 * world, dtype=np.int64)
    rc = comm.c.allgather(None, payload.ctypes.data, payload.nbytes, recv.ctypes.data)
    q.put((rank, rc, recv.tolist(), comm.rank, comm.world))
    dist.destroy_process_group()
    del C


def test_torch_comm_allgather_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    want = [0, 1, 2, 3, 4, 0, 2, 4, 6, 8]
    for rank, rc, recv, r, w in res:
        assert rc == 0 and recv == want and w == 2 and r == rank
