"""CPU tests of the multi-GPU host logic: the static column
division and the shard planner of mrrr_stemr_dist (mrrr_plan_columns, host
code of libmrrr_b200.so), and the all-gather callback of the binding with
the payloads the protocol exchanges (the root grid's int32 counts, whose
byte count need not be a multiple of 8; the bracket exchange [lo | hi |
status, clusters] and its merge-by-owner rule), exercised over
torch.distributed with the gloo backend, world_size 2."""
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


def _plan(m, nr, free):
    return M.plan_columns(m, nr, free)


@pytest.mark.parametrize("m,nr", [(1000, 4), (20000, 8), (97, 3), (5, 8)])
def test_planner_without_boundaries_is_static(m, nr):
    cuts = _plan(m, nr, [0] * (m + 1))
    assert cuts == [min(r * ((m + nr - 1) // nr), m) for r in range(nr + 1)]


def test_planner_moves_to_nearest_boundary_within_slack():
    m, nr = 4000, 4           # epp 1000, slack 25
    free = [0] * (m + 1)
    free[1010] = 1            # 10 right of cut 1
    free[1990] = free[2012] = 1   # cut 2: 10 left beats 12 right
    free[2960] = 1            # 40 left of cut 3: beyond the slack
    cuts = _plan(m, nr, free)
    assert cuts == [0, 1010, 1990, 3000, 4000]
    free[2990] = free[3010] = 1   # equidistant: ties go to the left
    assert _plan(m, nr, free)[3] == 2990


def test_planner_bound_on_shares():
    """Random boundary patterns: cuts are monotone, move at most epp/40, and
    every share fits the capacity epp + epp/20 the binding allocates."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        nr = int(rng.integers(2, 9))
        m = int(rng.integers(nr, 5000))
        free = list((rng.random(m + 1) < rng.choice([0.001, 0.01, 0.2])).astype(int))
        cuts = _plan(m, nr, free)
        epp = (m + nr - 1) // nr
        assert cuts[0] == 0 and cuts[-1] == m
        assert all(cuts[r] <= cuts[r + 1] for r in range(nr))
        for r in range(1, nr):
            st = min(r * epp, m)
            assert abs(cuts[r] - st) <= epp // 40
            assert cuts[r] == st or free[cuts[r]]
        assert max(cuts[r + 1] - cuts[r] for r in range(nr)) <= M.dist_capacity(m, nr)


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


def _worker_exchange(rank, world, port, out):
    """The protocol's two payload kinds through the binding's callback."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cb = M.torch_allgather(device="cpu")
        # (1) root grid counts: gp int32 per rank (gp odd: 4 * gp bytes is not a multiple of 8)
        gp = 5
        send = (C.c_int32 * gp)(*[1000 * rank + k for k in range(gp)])
        recv = (C.c_int32 * (gp * world))()
        rc1 = cb(None, C.addressof(send), C.addressof(recv), gp * 4, None)
        # (2) bracket exchange: [lo (ns) | hi (ns) | status, clusters] per rank,
        # then every rank merges slot q from its owner's part
        ns = 6
        owner = [0, 0, 0, 1, 1, 1]
        lo = [float(10 * rank + q) for q in range(ns)]
        hi = [float(10 * rank + q) + 0.5 for q in range(ns)]
        payload = lo + hi + [float(rank == 1) * 2.0, 7.0]
        xs = (C.c_double * len(payload))(*payload)
        xr = (C.c_double * (len(payload) * world))()
        rc2 = cb(None, C.addressof(xs), C.addressof(xr), len(payload) * 8, None)
        stride = 2 * ns + 2
        merged_lo = [xr[owner[q] * stride + q] for q in range(ns)]
        merged_hi = [xr[owner[q] * stride + ns + q] for q in range(ns)]
        status = [int(xr[r * stride + 2 * ns]) for r in range(world)]
        ncl = [int(xr[r * stride + 2 * ns + 1]) for r in range(world)]
        out[rank] = (rc1, list(recv), rc2, merged_lo, merged_hi, status, ncl)
    finally:
        dist.destroy_process_group()


def test_exchange_payloads_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_exchange, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        rc1, counts, rc2, mlo, mhi, status, ncl = out[r]
        assert rc1 == 0 and rc2 == 0
        assert counts == [0, 1, 2, 3, 4, 1000, 1001, 1002, 1003, 1004]
        # every rank ends with the same merged brackets: owners' values
        assert mlo == [0.0, 1.0, 2.0, 13.0, 14.0, 15.0]
        assert mhi == [0.5, 1.5, 2.5, 13.5, 14.5, 15.5]
        # the status word of rank 1 reaches rank 0 (worst code = 2 on both)
        assert status == [0, 2] and max(status) == 2
        assert ncl == [7, 7]


def _worker_uid(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        payload = bytes((7 * k + 1) % 256 for k in range(128)) if rank == 0 else bytes(range(128))
        out[rank] = M.broadcast_bytes(payload, rank)
    finally:
        dist.destroy_process_group()


def test_nccl_unique_id_bootstrap_gloo_world2():
    """NcclComm's bootstrap: every rank ends with rank 0's 128 ncclUniqueId
    bytes (zero bytes included), whatever it held before."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_uid, args=(world, port, out), nprocs=world, join=True)
    expect = bytes((7 * k + 1) % 256 for k in range(128))
    assert out[0] == expect and out[1] == expect
