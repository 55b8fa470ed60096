"""GPU edge cases and the paths the BASELINE configs never reach (VERDICT r01
"weak" 1): the Sturm counts of the bisection kernels against the oracle's,
integer for integer (mrrr_negcount); the qd safe path and the shift nudge,
forced through the diagnostic switches MRRR_FORCE_SAFE / MRRR_FORCE_NUDGE;
inputs scaled by 2^+-1000 (the library scales by an exact power of two, so
the results must scale bit for bit); a graded matrix; an off-diagonal exactly
at the split threshold eps ||T||_1 (reading 1/16: split iff |e_i| <= eps
||T||_1) and one ulp above; an INDEX range cutting exactly degenerate glued
groups; VALUE endpoints on eigenvalues (reading 15).  Everything goes through
the C ABI of libmrrr_b200.so and is compared with the oracle (oracle/).
"""
import os

import numpy as np
import pytest

from helpers import EPS, check_accuracy, residuals, tnorm1
from paper_1205_2107_b200 import workloads as W
from test_gpu_parity import compare, gpu_solve

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests (no CPU fallback exists)")
    return torch


@pytest.fixture(scope="module")
def P():
    import paper_1205_2107_b200 as P
    P.mrrr.lib()
    return P


def dense_ldl(D, LLD):
    """Eigenvalues of L D L^T (tridiagonal: diag D_i + LLD_{i-1}, offdiag L_i D_i)
    for the shift filter (numpy; test side only)."""
    n = len(D)
    L = np.sqrt(np.abs(LLD / D[:-1]))  # |L_i|: only |offdiag| matters for eigenvalues
    off = L * np.abs(D[:-1])
    diag = D.copy()
    diag[1:] += LLD
    A = np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)
    return np.linalg.eigvalsh(A)


ROOTS = {
    "random_1500": lambda: W.random_uniform(1500, 3),
    "one_two_one_600": lambda: W.one_two_one(600),
    "clement_500": lambda: W.clement(500),
    "wilkinson_301": lambda: W.wilkinson(301),
}


@pytest.mark.parametrize("name", list(ROOTS))
def test_negcount_bit_exact(torch_cuda, P, oracle_mod, name):
    """GPU counts (mode 0: the projective sweep of k_grid; mode 1: the qd safe
    path; mode 2: the twisted count of k_refine_warp, reading 32) equal the
    oracle's O6 count for shifts farther than 1e-9 |mu| from every eigenvalue
    of the representation (closer, the evaluation orders may legitimately
    round to different sides).  Includes
    dyadic grid shifts -- the root grid's points, which on structured inputs
    hit exact zero pivots (the oracle's NaN re-sweep; counted below)."""
    torch = torch_cuda
    d, e = ROOTS[name]()
    D, L, sigma = oracle_mod.root_rrr(d, e, side=1, perturb=1, seed=0x1205210700000000)
    LLD = L * L * D[:-1]
    lam = dense_ldl(D, LLD)
    hi0 = lam[-1] * 1.01 + 1e-12
    rng = np.random.default_rng(11)
    mus = np.concatenate([rng.uniform(0.0, hi0, 3000),
                          hi0 * np.arange(1, 1024) / 1024.0,     # dyadic grid points
                          lam[::7] * (1 + 1e-6), lam[::11] * (1 - 1e-6)])
    dist = np.min(np.abs(mus[:, None] - lam[None, :]), axis=1)
    keep = dist > 1e-9 * np.abs(mus)
    mus = mus[keep]
    ref, zero_piv = [], 0
    for mu in mus:
        c, rs = oracle_mod.negcount(D, None, mu, LLD=LLD, return_resweep=True)
        ref.append(c)
        zero_piv += rs
    ref = np.array(ref)
    Dt, Lt, mt = (torch.tensor(x, device="cuda") for x in (D, LLD, mus))
    for mode in (0, 1, 2):
        got = P.mrrr.negcount(Dt, Lt, mt, mode=mode).cpu().numpy()
        bad = np.nonzero(got != ref)[0]
        assert len(bad) == 0, (mode, len(bad), zero_piv, mus[bad[:5]], got[bad[:5]], ref[bad[:5]])
    # the count equals the dense count too (independent of both sides)
    assert np.array_equal(ref, np.searchsorted(lam, mus, side="left"))


def test_negcount_exact_zero_pivot(torch_cuda, P, oracle_mod):
    """A shift that makes a pivot exactly zero: T = 1-2-1 (D = 2, ...) with mu
    = 2 on the UNSHIFTED factorization of 2I + offdiag (D_0 = 2, so D+_0 = 0
    at mu = 2).  mu = 2 is an eigenvalue of the leading 1x1 block, not of the
    whole matrix for even n, so the count is well defined; the oracle takes
    its NaN re-sweep, the projective sweep passes the zero as projective
    infinity, and both must give the count."""
    torch = torch_cuda
    n = 64
    d, e = W.one_two_one(n)
    # exact LDL^T of T (no shift): D_0 = 2, D_{i+1} = 2 - 1/D_i, L_i = 1/D_i
    D = np.zeros(n)
    Lv = np.zeros(n - 1)
    D[0] = 2.0
    for i in range(n - 1):
        Lv[i] = 1.0 / D[i]
        D[i + 1] = 2.0 - Lv[i]
    LLD = Lv * Lv * D[:-1]
    mus = np.array([2.0, 1.0, 3.0, 0.5])
    ref = [oracle_mod.negcount(D, None, mu, LLD=LLD, return_resweep=True) for mu in mus]
    assert ref[0][1], "mu = 2 must hit an exact zero pivot in the oracle"
    Dt, Lt, mt = (torch.tensor(x, device="cuda") for x in (D, LLD, mus))
    for mode in (0, 1, 2):
        got = P.mrrr.negcount(Dt, Lt, mt, mode=mode).cpu().numpy()
        assert list(got) == [r[0] for r in ref], (mode, got, ref)
    k = np.arange(1, n + 1)
    lam = 2 - 2 * np.cos(k * np.pi / (n + 1))
    assert [r[0] for r in ref] == list(np.searchsorted(lam, mus))


@pytest.mark.parametrize("env,stat", [("MRRR_FORCE_SAFE", "safe_resweeps"),
                                      ("MRRR_FORCE_NUDGE", "vec_nudges")])
@pytest.mark.parametrize("case", ["random_700", "glued_12", "clement_300_idx"])
def test_forced_fallback_paths(torch_cuda, P, oracle_mod, monkeypatch, env, stat, case):
    """The qd safe path of every Sturm sweep (MRRR_FORCE_SAFE: the grid, root
    interval and refinement kernels take negcount_qd_safe for every shift) and
    the vector kernels' shift nudge (MRRR_FORCE_NUDGE: every first twisted
    factorization is treated as failed, reading 25) are exercised in full
    solves: parity with the oracle and the accuracy contract hold, and the
    counters show the path ran."""
    kw = {}
    if case == "random_700":
        d, e = W.random_uniform(700, 4)
    elif case == "glued_12":
        d, e = W.glued_wilkinson(12)
    else:
        d, e = W.clement(300)
        kw = {"il": 1, "iu": 40}
    monkeypatch.setenv(env, "1")
    w, Z = gpu_solve(P, torch_cuda, d, e, **kw)
    st = P.last_stats()
    monkeypatch.delenv(env)
    assert st[stat] > 0, st
    wo, Zo = oracle_mod.stemr(d, e, **kw)
    compare(d, e, w, Z, wo, Zo, full_range=not kw)
    # switching back off restores the default path (the flag is per call)
    w2, Z2 = gpu_solve(P, torch_cuda, d, e, **kw)
    assert P.last_stats()[stat] == 0
    compare(d, e, w2, Z2, wo, Zo, full_range=not kw)


@pytest.mark.parametrize("k", [1000, -960, 37])
@pytest.mark.parametrize("case", ["random_500", "glued_10"])
def test_power_of_two_scaling(torch_cuda, P, case, k):
    """T 2^k: the library scales T by an exact power of two to ||T||_1 in
    [1, 2), so w(T 2^k) = 2^k w(T) and Z(T 2^k) = Z(T) bit
    for bit -- at 2^1000 (entries near 1e301) and 2^-960 (near 1e-289; the
    glue 1e-8 stays a normal number, which an exact scaling needs)."""
    d, e = W.random_uniform(500, 8) if case == "random_500" else W.glued_wilkinson(10)
    w0, Z0 = gpu_solve(P, torch_cuda, d, e)
    w1, Z1 = gpu_solve(P, torch_cuda, np.ldexp(d, k), np.ldexp(e, k))
    assert np.array_equal(w1, np.ldexp(w0, k))
    assert np.array_equal(Z1, Z0)


@pytest.mark.parametrize("rho,n", [(0.5, 45), (0.9, 300)])
def test_graded_matrix(torch_cuda, P, oracle_mod, rho, n):
    """Graded T: d_i = rho^i, e_i = 0.3 rho^(i+1/2) -- eigenvalues over 14
    decades, no split (e_{n-2} > eps ||T||_1)."""
    i = np.arange(n, dtype=np.float64)
    d = rho ** i
    e = 0.3 * rho ** (i[:-1] + 0.5)
    assert np.min(np.abs(e)) > EPS * tnorm1(d, e)
    w, Z = gpu_solve(P, torch_cuda, d, e)
    wo, Zo = oracle_mod.stemr(d, e)
    compare(d, e, w, Z, wo, Zo)
    mu, _ = oracle_mod.jacobi(np.diag(d) + np.diag(e, 1) + np.diag(e, -1)) if n <= 64 else (None, None)
    if mu is not None:
        assert np.max(np.abs(w - mu)) <= 4 * n * EPS * tnorm1(d, e)


@pytest.mark.parametrize("above", [False, True])
def test_split_threshold(torch_cuda, P, oracle_mod, above):
    """|e_i| = eps ||T||_1 splits (reading 16: <=), one ulp above does not;
    the GPU and the oracle take the same decision, and a split leaves the
    columns zero outside their block."""
    n, cut = 200, 100
    d, e = W.random_uniform(n, 12)
    d[cut] = d[cut + 1] = 0.0
    e[cut] = 0.0
    tn = oracle_mod.norms(d, e)[0]  # summed in the library's order: (|e_i-1| + |e_i|) + |d_i|
    e[cut] = EPS * tn
    if above:
        e[cut] = np.nextafter(e[cut], np.inf)
    assert oracle_mod.norms(d, e)[0] == tn  # rows cut, cut+1 are not the norm's row
    w, Z = gpu_solve(P, torch_cuda, d, e)
    wo, Zo = oracle_mod.stemr(d, e)
    compare(d, e, w, Z, wo, Zo)
    top = np.any(Z[:cut + 1] != 0, axis=0)
    bot = np.any(Z[cut + 1:] != 0, axis=0)
    if not above:
        assert not np.any(top & bot)  # every column lives in one block
        assert len(oracle_mod.split(d, e)) == 3
    else:
        assert len(oracle_mod.split(d, e)) == 2


@pytest.mark.parametrize("il,iu", [(21, 60), (33, 33), (5, 118)])
def test_index_range_cuts_degenerate_groups(torch_cuda, P, oracle_mod, il, iu):
    """Glued W21+ x 40: groups of 40 eigenvalues equal in fp64 (SURVEY [A1]).
    An INDEX range that cuts a group returns some orthonormal vectors of the
    group's invariant subspace: eigenvalues match the oracle, the residual and
    orthogonality hold, and every returned column lies in the span of the
    oracle's vectors of the whole groups it touches (subspace test)."""
    d, e = W.glued_wilkinson(40)
    n = len(d)
    w, Z = gpu_solve(P, torch_cuda, d, e, il=il, iu=iu)
    wo, _ = oracle_mod.stemr(d, e, il=il, iu=iu, vectors=False)
    assert len(w) == iu - il + 1
    assert np.max(np.abs(w - wo)) <= 4 * n * EPS * tnorm1(d, e)
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1, (res, orth)
    g0, g1 = (il - 1) // 40 * 40 + 1, (iu - 1) // 40 * 40 + 40
    _, Q = oracle_mod.stemr(d, e, il=g0, iu=g1)
    proj = Z - Q @ (Q.T @ Z)
    assert np.max(np.linalg.norm(proj, axis=0)) <= 1e-9


@pytest.mark.parametrize("vl,vu", [(-1.0, 3.0), (-5.0, -1.0), (-399.0, -391.0), (397.0, 399.0)])
def test_value_endpoints_on_eigenvalues(torch_cuda, P, oracle_mod, vl, vu):
    """Clement n=400: eigenvalues +-1, +-3, ..., +-399 (closed form).  VALUE
    endpoints placed ON eigenvalues (reading 15: indices N(vl)+1 .. N(vu) by
    Sturm counts of T, i.e. (vl, vu] up to the rounding of the count at an
    eigenvalue): the GPU returns the same index set as the oracle, the
    eigenvalues match the closed form, and the vectors pass the contract."""
    n = 400
    d, e = W.clement(n)
    w, Z = gpu_solve(P, torch_cuda, d, e, vl=vl, vu=vu)
    wo, Zo = oracle_mod.stemr(d, e, vl=vl, vu=vu)
    assert len(w) == len(wo), (len(w), len(wo), w, wo)
    compare(d, e, w, Z, wo, Zo, full_range=False)
    lam = 2.0 * np.arange(1, n + 1) - n - 1
    k0 = int(np.searchsorted(lam, w[0] - 0.5)) if len(w) else 0
    assert np.max(np.abs(w - lam[k0:k0 + len(w)])) <= 4 * n * EPS * tnorm1(d, e)
    # the set is contiguous and lies in [vl, vu] up to the counting tie
    assert lam[k0] >= vl - 1e-9 and lam[k0 + len(w) - 1] <= vu + 1e-9


@pytest.mark.parametrize("case", ["random_3000", "glued_40", "clement_2000_idx"])
def test_workspace_bound(torch_cuda, P, case):
    """mrrr_workspace_bytes(n, k) bounds the workspace a call uses, apart from
    the cluster nodes' child representations (16 n B per slot, reported as
    pool_bytes: recycled, so at most one slot per node); include/mrrr.h."""
    kw = {}
    if case == "random_3000":
        d, e = W.random_uniform(3000, 2)
    elif case == "glued_40":
        d, e = W.glued_wilkinson(40)
    else:
        d, e = W.clement(2000)
        kw = {"il": 1, "iu": 500}
    gpu_solve(P, torch_cuda, d, e, **kw)
    st = P.last_stats()
    n, k = len(d), (kw["iu"] - kw["il"] + 1 if kw else len(d))
    bound = P.mrrr.lib().mrrr_workspace_bytes(n, k)
    assert st["nodes"] == 0 or 16 * n <= st["pool_bytes"] <= 16 * n * st["nodes"]
    assert 0 < st["workspace_bytes"] - st["pool_bytes"] <= bound, (st["workspace_bytes"], st["pool_bytes"], bound)


def test_scratch_cap_and_pool_recycling(torch_cuda, P):
    """mrrr_opts_t.scratch_gb bounds the two large scratch areas: at 0.25 GB
    (random n=20000) the vector pieces hold <= 781 eigenvectors and the
    cluster steps run in groups of <= 86 clusters -- more launches, less
    workspace, and not a bit of difference in w or Z (each eigenpair's RQC and
    each cluster's step depend on their own data only).  The child
    representation slots are recycled: fewer slots than tree nodes."""
    d, e, _ = W.make("random_20000")
    n = len(d)
    w1, Z1 = gpu_solve(P, torch_cuda, d, e)
    s1 = P.last_stats()
    P.trim_workspace()
    w2, Z2 = gpu_solve(P, torch_cuda, d, e, opts=P.default_opts(scratch_gb=0.25))
    s2 = P.last_stats()
    P.trim_workspace()
    assert np.array_equal(w1, w2) and np.array_equal(Z1, Z2)
    assert s2["kernel_launches"] > s1["kernel_launches"]
    assert s2["workspace_bytes"] < s1["workspace_bytes"]
    assert s1["nodes"] == s2["nodes"] and s1["nodes"] > 1000
    for s in (s1, s2):
        assert 16 * n <= s["pool_bytes"] < 16 * n * s["nodes"]


@pytest.mark.parametrize("root_m", ["1", "2", "4"])
@pytest.mark.parametrize("n", [3, 5, 7, 9, 11, 21, 101, 1001])
def test_zero_diagonal_exact_zero_eigenvalue(torch_cuda, P, oracle_mod, monkeypatch, n, root_m):
    """d = 0, e = 1 (odd n: eigenvalue 0 exactly, its vector zero at every odd
    row).  With some root brackets the eigenvalue sits within rounding of a
    bracket end; the RQC step then overshoots the end by an ulp or two, which
    reading 24 (amended) clamps to the end instead of bisecting -- bisection
    halved every later correction and the stagnation test stopped the lane at
    ~1e-10 (residual 4e4x the bound at n = 3 and 21).  The root refinement's
    shifts per lane (MRRR_RW_ROOT_M) change the brackets."""
    monkeypatch.setenv("MRRR_RW_ROOT_M", root_m)
    d, e = np.zeros(n), np.ones(n - 1)
    w, Z = gpu_solve(P, torch_cuda, d, e)
    lam = np.sort(2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    assert np.max(np.abs(w - lam)) <= 4 * n * EPS * tnorm1(d, e)
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1, (res, orth)


def test_rqc_histogram(torch_cuda, P):
    """mrrr_get_rqc_histogram: every eigenvector of the tree's vector kernels is
    counted once, under the number of twisted factorizations its RQC took; the
    weighted sum is the call's factorization count (no fallback on this input);
    a values-only solve counts nothing."""
    torch = torch_cuda
    d, e = W.random_uniform(3000, 4)
    dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    w, Z = P.stemr(dt, et)
    st = P.last_stats()
    h = P.rqc_histogram()
    assert len(h) == 16 and h[0] == 0
    assert sum(h) == 3000
    assert st["rqc_fallbacks"] == 0
    assert sum(k * c for k, c in enumerate(h)) == st["rqc_iters"]
    assert max(k for k, c in enumerate(h) if c) <= 10  # reading 10: at most 10 factorizations
    w, _ = P.stemr(dt, et, vectors=False)
    assert sum(P.rqc_histogram()) == 0


@pytest.mark.parametrize("case", ["random_3000", "glued_40", "clement_2000"])
def test_rqc_previous_correction_stop(torch_cuda, P, monkeypatch, case):
    """DESIGN.md reading 33 (GPU only): the RQC stops at a factorization whose
    shift was reached by a Rayleigh-quotient step of at most 2^-31 |lambda|.
    With the rule and without it (MRRR_RQC_PREV_TOL=0: reading 10 alone, as
    the oracle iterates) the eigenvalues agree to rounding level, both meet the
    residual / orthogonality contract, and the rule never costs a factorization."""
    d, e = {"random_3000": lambda: W.random_uniform(3000, 4), "glued_40": lambda: W.glued_wilkinson(40),
            "clement_2000": lambda: W.clement(2000)}[case]()
    w1, Z1 = gpu_solve(P, torch_cuda, d, e)
    h1, st1 = P.rqc_histogram(), P.last_stats()
    monkeypatch.setenv("MRRR_RQC_PREV_TOL", "0")
    w0, Z0 = gpu_solve(P, torch_cuda, d, e)
    h0, st0 = P.rqc_histogram(), P.last_stats()
    monkeypatch.delenv("MRRR_RQC_PREV_TOL")
    w2, Z2 = gpu_solve(P, torch_cuda, d, e)  # the default is restored for the tests that follow
    assert np.array_equal(w1, w2) and np.array_equal(Z1, Z2)
    n, tn = len(d), tnorm1(d, e)
    assert np.max(np.abs(w1 - w0)) <= 8 * EPS * tn
    for w, Z in ((w1, Z1), (w0, Z0)):
        res, orth = check_accuracy(d, e, w, Z)
        assert res <= 1 and orth <= 1, (res, orth)
    assert sum(h1) == sum(h0) == n
    assert st1["rqc_iters"] <= st0["rqc_iters"]
    assert max(k for k, c in enumerate(h1) if c) <= max(k for k, c in enumerate(h0) if c)
