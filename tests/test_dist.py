"""CPU tests of the multi-GPU host logic: the static column
division of mrrr_stemr_dist and the all-gather callback of the binding,
exercised over torch.distributed with the gloo backend, world_size 2."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1205_2107_b200 import mrrr as M


@pytest.mark.parametrize("m,nranks", [(1, 1), (7, 2), (20000, 8), (5, 8), (100000, 3), (0, 4)])
def test_shard_columns_partition(m, nranks):
    """Shards are contiguous, disjoint, cover [0, m) in rank order and differ
    in size by at most ceil(m / nranks) - floor(m / nranks) except the tail."""
    prev = 0
    epp = (m + nranks - 1) // nranks
    for r in range(nranks):
        c0, c1 = M.shard_columns(m, nranks, r)
        assert c0 == prev and c0 <= c1 <= m
        assert c1 - c0 <= epp
        prev = c1
    assert prev == m


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = 11
        epp = (m + world - 1) // world
        c0, c1 = M.shard_columns(m, world, rank)
        # this rank's padded part of w (as the library lays it out)
        send = (C.c_double * epp)(*([100.0 * rank + k for k in range(c1 - c0)] + [0.0] * (epp - (c1 - c0))))
        recv = (C.c_double * (epp * world))()
        cb = M.torch_allgather(device="cpu")
        rc = cb(None, C.addressof(send), C.addressof(recv), epp * 8, None)
        out[rank] = (rc, list(recv))
    finally:
        dist.destroy_process_group()


def test_allgather_callback_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    m = 11
    epp = (m + world - 1) // world
    expect = []
    for r in range(world):
        c0, c1 = M.shard_columns(m, world, r)
        expect += [100.0 * r + k for k in range(c1 - c0)] + [0.0] * (epp - (c1 - c0))
    for r in range(world):
        rc, recv = out[r]
        assert rc == 0
        assert recv == expect
