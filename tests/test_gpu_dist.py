"""GPU tests of mrrr_stemr_dist on one GPU: P virtual ranks run one after
another; the only collective (the all-gather of w) is replaced by a callback
that places this rank's part (nothing else is exchanged), and the test
assembles w and Z from the P calls.  Checks: every column is computed by
exactly one rank, the assembled spectrum matches the oracle, and the
assembled Z -- whose columns come from different ranks, i.e. across shard
boundaries through clusters shared by several ranks -- is orthogonal and
accurate (BASELINE tolerances)."""
import ctypes as C

import numpy as np
import pytest

from helpers import EPS, check_accuracy, dk_comparable, residuals, tnorm1, vec_diff_signfree
from paper_1205_2107_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch


def local_allgather(rank, nranks=1):
    """Stand-in for the all-gather on one process: recv[rank part] <- send;
    the other ranks' parts read -inf (they are never used for own columns;
    the library's monotone fix is a running max)."""
    import torch
    from paper_1205_2107_b200 import mrrr as M

    def fn(ctx, send, recv, nbytes, stream):
        with torch.cuda.stream(M._ext_stream(stream)):  # on the library's stream
            st = torch.as_tensor(M._DevBuf(send, nbytes), device="cuda")
            allr = torch.as_tensor(M._DevBuf(recv, nbytes * nranks), device="cuda")
            allr.fill_(float("-inf"))
            allr[rank * (nbytes // 8):(rank + 1) * (nbytes // 8)].copy_(st)
        return 0
    return M.ALLGATHER_FN(fn)


def run_virtual(torch, d, e, nranks, **kw):
    import paper_1205_2107_b200 as P
    n = len(d)
    dt = torch.tensor(d, device="cuda")
    et = torch.tensor(e if len(e) else np.zeros(1), device="cuda")
    parts = []
    for r in range(nranks):
        cb = local_allgather(r, nranks)
        w_all, Zl, c0 = P.stemr_dist(dt, et, rank=r, nranks=nranks, allgather=cb, **kw)
        torch.cuda.synchronize()
        m = w_all.shape[0]
        cs0, c1 = P.shard_columns(m, nranks, r)
        assert c0 == cs0
        if Zl is not None:
            assert Zl.shape[1] == c1 - c0
        parts.append((c0, c1, w_all.cpu().numpy()[c0:c1].copy(),
                      Zl.cpu().numpy().copy() if Zl is not None else None))
    m = parts[-1][1]
    w = np.concatenate([p[2] for p in parts])
    Z = np.concatenate([p[3] for p in parts], axis=1) if parts[0][3] is not None else None
    assert len(w) == m
    return w, Z


CASES = {
    "random_1500": (lambda: W.random_uniform(1500, 4), {}),
    "glued_40": (lambda: W.glued_wilkinson(40), {}),
    "one_two_one_900": (lambda: W.one_two_one(900), {}),
    "clement_1200_idx": (lambda: W.clement(1200), {"il": 1, "iu": 300}),
    "random_1000_idx": (lambda: W.random_uniform(1000, 2), {"il": 201, "iu": 777}),
}


@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("name", list(CASES))
def test_dist_virtual_ranks(torch_cuda, oracle_mod, name, nranks):
    mk, kw = CASES[name]
    d, e = mk()
    n = len(d)
    w, Z = run_virtual(torch_cuda, d, e, nranks, **kw)
    wo, Zo = oracle_mod.stemr(d, e, **kw)
    assert len(w) == len(wo)
    assert np.all(np.diff(w) >= 0)
    assert np.max(np.abs(w - wo)) <= 4 * n * EPS * tnorm1(d, e)
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1, (res, orth)
    ok = dk_comparable(wo, residuals(d, e, w, Z), residuals(d, e, wo, Zo))
    if ok.any():
        assert np.max(vec_diff_signfree(Z[:, ok], Zo[:, ok])) <= 1e-9


def test_dist_values_only(torch_cuda, oracle_mod):
    d, e = W.random_uniform(800, 5)
    w, _ = run_virtual(torch_cuda, d, e, 4, vectors=False)
    wo, _ = oracle_mod.stemr(d, e, vectors=False)
    assert np.max(np.abs(w - wo)) <= 4 * len(d) * EPS * tnorm1(d, e)


def test_dist_single_rank_equals_stemr(torch_cuda):
    import paper_1205_2107_b200 as P
    torch = torch_cuda
    d, e = W.random_uniform(700, 6)
    dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    w1, Z1 = P.stemr(dt, et)
    w2, Z2, c0 = P.stemr_dist(dt, et, rank=0, nranks=1, allgather=local_allgather(0))
    assert c0 == 0
    assert torch.equal(w1, w2) and torch.equal(Z1, Z2)


def test_dist_argument_errors(torch_cuda):
    import paper_1205_2107_b200 as P
    torch = torch_cuda
    d, e = W.random_uniform(50, 0)
    dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    with pytest.raises(P.mrrr.MrrrError) as ex:
        P.stemr_dist(dt, et, rank=3, nranks=2, allgather=local_allgather(0))
    assert ex.value.code == -9
    with pytest.raises(P.mrrr.MrrrError) as ex:
        P.stemr_dist(dt, et, rank=0, nranks=0, allgather=local_allgather(0))
    assert ex.value.code == -10
