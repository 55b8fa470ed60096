"""GPU tests of mrrr_stemr_dist on one GPU: P virtual ranks (tests/vranks.py:
P host threads, each with its own stream, exchanging through a host-side
all-gather) run the whole protocol of DESIGN.md §6 -- split root grid and
root bisection with their gathers, the shard planner, the per-level bracket
exchange of shared clusters (type-3 tasks), the final gather
of w, and the status word.  Checks: every column is computed by exactly one
rank, the shares respect the planner's bound, w is identical on every rank,
the assembled spectrum matches the oracle, and the assembled Z -- whose
columns come from different ranks, i.e. across shard boundaries through
clusters shared by several ranks -- is orthogonal and accurate (BASELINE
tolerances); a failure on one rank makes every rank return the same code
(no rank hangs)."""
import numpy as np
import pytest

from helpers import EPS, check_accuracy, dk_comparable, residuals, tnorm1, vec_diff_signfree
from paper_1205_2107_b200 import workloads as W
from vranks import VirtualRanks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch


def run_virtual(torch, d, e, nranks, vectors=True, **kw):
    from paper_1205_2107_b200 import mrrr as M
    out = VirtualRanks(nranks).run(d, e, vectors=vectors, **kw)
    for r, o in enumerate(out):
        assert o[0] == 0, (r, o[0], o[1])
    m = out[0][1].shape[0]
    w0 = out[0][1].cpu().numpy()
    cap = M.dist_capacity(m if "il" in kw else len(d), nranks)
    prev = 0
    w_parts, Z_parts = [], []
    for r, (_, w_all, Zl, c0, st) in enumerate(out):
        assert np.array_equal(w_all.cpu().numpy(), w0)  # every rank holds the same w
        ml = Zl.shape[1] if Zl is not None else None
        if vectors:
            assert c0 == prev
            assert ml <= cap
            Z_parts.append(Zl.cpu().numpy())
            prev = c0 + ml
    if vectors:
        assert prev == m  # the shares tile [0, m)
    Z = np.concatenate(Z_parts, axis=1) if vectors else None
    return w0, Z, out


CASES = {
    "random_1500": (lambda: W.random_uniform(1500, 4), {}),
    "glued_40": (lambda: W.glued_wilkinson(40), {}),
    "one_two_one_900": (lambda: W.one_two_one(900), {}),
    "clement_1200_idx": (lambda: W.clement(1200), {"il": 1, "iu": 300}),
    "random_1000_idx": (lambda: W.random_uniform(1000, 2), {"il": 201, "iu": 777}),
    "split_3blocks": (None, {}),
}


def split_matrix():
    d1, e1 = W.random_uniform(300, 11)
    d2, e2 = W.one_two_one(250)
    d3, e3 = W.wilkinson(21)
    d = np.concatenate([d1, d2 - 1.0, d3 * 0.2])
    e = np.concatenate([e1, [0.0], e2, [0.0], e3 * 0.2])
    return d, e


@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("name", list(CASES))
def test_dist_virtual_ranks(torch_cuda, oracle_mod, name, nranks):
    mk, kw = CASES[name]
    d, e = mk() if mk else split_matrix()
    n = len(d)
    w, Z, _ = run_virtual(torch_cuda, d, e, nranks, **kw)
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
    w, _, _ = run_virtual(torch_cuda, d, e, 4, vectors=False)
    wo, _ = oracle_mod.stemr(d, e, vectors=False)
    assert np.max(np.abs(w - wo)) <= 4 * len(d) * EPS * tnorm1(d, e)


def test_dist_ranks_match_single_gpu(torch_cuda):
    """The split root work, the exchanges and the split refinement change no
    bit: the P-rank eigenpairs equal the single-GPU solve's (each member's
    refinement depends on its rank-invariant work item alone)."""
    import paper_1205_2107_b200 as P
    torch = torch_cuda
    d, e = W.random_uniform(2500, 6)
    dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    w1, Z1 = P.stemr(dt, et)
    w1, Z1 = w1.cpu().numpy(), Z1.cpu().numpy()
    for nr in (2, 5):
        w, Z, _ = run_virtual(torch, d, e, nr)
        assert np.array_equal(w, w1)
        assert np.array_equal(Z, Z1)


def test_dist_shard_planner_moves_cuts(torch_cuda):
    """The planner moves cuts only to root-cluster boundaries within epp/40:
    on 1-2-1 n=900 (three root clusters, SURVEY [A2]) the shares stay within
    the bound and some cut differs from the static one or sits on a
    boundary the planner could not move."""
    from paper_1205_2107_b200 import mrrr as M
    d, e = W.one_two_one(900)
    _, _, out = run_virtual(torch_cuda, d, e, 4)
    cuts = [o[3] for o in out] + [900]
    epp = 225
    for r in range(1, 4):
        assert abs(cuts[r] - r * epp) <= epp // 40
    assert max(cuts[r + 1] - cuts[r] for r in range(4)) <= M.dist_capacity(900, 4)


def test_dist_error_on_one_rank(torch_cuda, monkeypatch):
    """MRRR_TEST_FAIL_RANK=1: rank 1 alone fails at tree level 0 (a child-RRR
    error); the status word of the level's exchange makes EVERY rank return
    that code at the same collective -- none is left waiting."""
    monkeypatch.setenv("MRRR_TEST_FAIL_RANK", "1")
    monkeypatch.setenv("MRRR_TEST_FAIL_LEVEL", "0")
    d, e = W.random_uniform(1200, 7)
    out = VirtualRanks(3).run(d, e)
    assert [o[0] for o in out] == [2, 2, 2], out
    monkeypatch.delenv("MRRR_TEST_FAIL_RANK")
    w, Z, _ = run_virtual(torch_cuda, d, e, 3)  # the same ranks recover on the next call
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1


def test_dist_single_rank_equals_stemr(torch_cuda):
    import paper_1205_2107_b200 as P
    torch = torch_cuda
    d, e = W.random_uniform(700, 6)
    dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    w1, Z1 = P.stemr(dt, et)
    w2, Z2, c0 = P.stemr_dist(dt, et, rank=0, nranks=1, allgather=VirtualRanks(1).callback(0))
    assert c0 == 0
    assert torch.equal(w1, w2) and torch.equal(Z1, Z2)


def test_dist_argument_errors(torch_cuda):
    import paper_1205_2107_b200 as P
    torch = torch_cuda
    d, e = W.random_uniform(50, 0)
    dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    cb = VirtualRanks(1).callback(0)
    with pytest.raises(P.mrrr.MrrrError) as ex:
        P.stemr_dist(dt, et, rank=3, nranks=2, allgather=cb)
    assert ex.value.code == -9
    with pytest.raises(P.mrrr.MrrrError) as ex:
        P.stemr_dist(dt, et, rank=0, nranks=0, allgather=cb)
    assert ex.value.code == -10


def test_nccl_entry_single_rank(torch_cuda):
    """mrrr_stemr_nccl on a one-rank ncclComm_t (what one GPU can run): the
    library resolves NCCL itself, reads rank / size from the communicator and
    issues every all-gather of the protocol as ncclAllGather on the solve
    stream; the eigenpairs equal mrrr_stemr's bit for bit (with vectors, values
    only and an index range), and a communicator of another device is refused."""
    import paper_1205_2107_b200 as P
    torch = torch_cuda
    comm = P.NcclComm("cuda:0", rank=0, nranks=1)
    try:
        for n, seed, kw in [(700, 6, {}), (1500, 2, {"il": 100, "iu": 900}), (900, 1, {"vectors": False})]:
            d, e = W.random_uniform(n, seed)
            dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
            w1, Z1 = P.stemr(dt, et, **kw)
            w2, Z2, c0 = P.stemr_nccl(dt, et, comm, **kw)
            assert c0 == 0
            assert torch.equal(w1, w2)
            assert (Z1 is None and Z2 is None) or torch.equal(Z1, Z2)
        assert P.last_stats()["kernel_launches"] > 0
    finally:
        comm.destroy()
    with pytest.raises(P.mrrr.MrrrError) as ex:
        P.stemr_nccl(dt, et, comm)  # destroyed: NULL handle
    assert ex.value.code == -9
