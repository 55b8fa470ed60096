"""Virtual ranks (test tooling): the P ranks of mrrr_stemr_dist as P host
threads on ONE GPU, each with its own CUDA stream, exchanging through a
host-side all-gather.

The all-gather callback of rank r: synchronise the library's stream (its
send buffer is complete), publish the send pointer, wait at a host barrier,
copy every rank's send buffer into its own recv buffer (device to device, on
the library's stream), synchronise, and wait at a second barrier before
returning (no rank overwrites a send buffer before every rank has copied
it).  Only HOST threads ever wait for each other; no kernel of one rank
waits on another rank (B200_PROFILING.md: ranks whose kernels wait on each
other must not share a GPU).

``timed=True`` also serialises the ranks' GPU work between collectives with
a lock (each rank runs its phase alone on the GPU, synchronised at both
ends, its device-side vector pieces included) and records per-phase wall
times, so that a P-GPU step can be projected as sum over phases of
max over ranks (tools/virtual_scaling.py)."""
from __future__ import annotations

import threading
import time

import torch

from paper_1205_2107_b200 import mrrr as M


class _Worker:
    """A persistent host thread (its library workspace, streams and events
    stay warm across calls, as a real rank's would)."""

    def __init__(self):
        import queue
        self.q = queue.Queue()
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        while True:
            fn, done = self.q.get()
            if fn is None:
                return
            try:
                fn()
            finally:
                done.set()

    def submit(self, fn):
        done = threading.Event()
        self.q.put((fn, done))
        return done


_POOL = []


def _workers(n):
    while len(_POOL) < n:
        _POOL.append(_Worker())
    return _POOL[:n]


class VirtualRanks:
    def __init__(self, nranks: int, timed: bool = False, timeout: float = 600.0):
        self.n = nranks
        self.bar = threading.Barrier(nranks, timeout=timeout)
        self.send = [None] * nranks
        self.timed = timed
        self.gpu = threading.Lock()
        self.phase_ms = [[] for _ in range(nranks)]
        self._t0 = [None] * nranks
        self.errors = []

    def _begin(self, rank):
        if self.timed:
            self.gpu.acquire()
            torch.cuda.synchronize()
            self._t0[rank] = time.perf_counter()

    def _end(self, rank):
        if self.timed:
            torch.cuda.synchronize()  # the rank's side-stream vector pieces too
            self.phase_ms[rank].append(1e3 * (time.perf_counter() - self._t0[rank]))
            self.gpu.release()

    def callback(self, rank: int):
        def fn(ctx, send, recv, nbytes, stream):
            try:
                st = M._ext_stream(stream)
                st.synchronize()
                self._end(rank)
                self.send[rank] = (send, nbytes)
                self.bar.wait()
                with torch.cuda.stream(st):
                    rv = torch.as_tensor(M._DevBuf(recv, nbytes * self.n, "|u1"), device="cuda")
                    for r in range(self.n):
                        sp, nb = self.send[r]
                        assert nb == nbytes, (nb, nbytes)
                        sv = torch.as_tensor(M._DevBuf(sp, nb, "|u1"), device="cuda")
                        rv[r * nbytes:(r + 1) * nbytes].copy_(sv)
                st.synchronize()
                self.bar.wait()
                self._begin(rank)
                return 0
            except Exception as ex:  # broken barrier, timeout: reported as MRRR_ERR_COMM
                self.errors.append(repr(ex))
                self.bar.abort()
                return 1
        return M.ALLGATHER_FN(fn)

    def run(self, d, e, **kw):
        """Run all ranks; returns per rank (rc, w_all, Z_local, col_begin) or
        the exception; plus the per-phase times when timed."""
        import paper_1205_2107_b200 as P
        dt = torch.tensor(d, device="cuda")
        et = torch.tensor(e if len(e) else [0.0], device="cuda", dtype=torch.float64)
        out = [None] * self.n
        cbs = [self.callback(r) for r in range(self.n)]

        def work(r):
            stream = torch.cuda.Stream()
            try:
                self._begin(r)
                with torch.cuda.stream(stream):
                    w_all, Zl, c0 = P.stemr_dist(dt, et, rank=r, nranks=self.n, allgather=cbs[r],
                                                 stream=stream, **kw)
                stream.synchronize()
                self._end(r)
                out[r] = (0, w_all, Zl, c0, P.last_stats())
            except M.MrrrError as ex:
                if self.timed and self.gpu.locked():
                    try:
                        self.gpu.release()
                    except RuntimeError:
                        pass
                out[r] = (ex.code, None, None, None, None)
            except Exception as ex:  # noqa: BLE001
                out[r] = (-999, repr(ex), None, None, None)

        done = [wk.submit(lambda r=r: work(r)) for r, wk in enumerate(_workers(self.n))]
        for ev in done:
            assert ev.wait(timeout=900), "a virtual rank hung"
        return out
