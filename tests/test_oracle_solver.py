"""End-to-end pins of the oracle solver against closed forms, brute-force
Jacobi, the Weyl bound, exact invariants, independent Sturm counts and LAPACK
(scipy) -- CPU only."""
import numpy as np
import pytest
import scipy.linalg as sl

from helpers import (EPS, check_accuracy, dk_comparable, residuals, sturm_placement, tnorm1,
                     vec_diff_signfree)
from paper_1205_2107_b200 import workloads as W


def dense_T(d, e):
    return np.diag(d) + np.diag(e, 1) + np.diag(e, -1)


def test_config1_one_two_one_closed_form(oracle_mod):
    """configs[0]: 1-2-1 n=2000, lambda_k = 2-2cos(k pi/2001) and
    z_k(i) = (-1)^i sqrt(2/2001) sin(i k pi/2001) (reading 23)."""
    n = 2000
    d, e = W.one_two_one(n)
    w, Z = oracle_mod.stemr(d, e)
    tn = tnorm1(d, e)
    k = np.arange(1, n + 1)
    lam = 2 - 2 * np.cos(k * np.pi / (n + 1))
    assert np.max(np.abs(w - lam)) <= 4 * n * EPS * tn
    i = np.arange(1, n + 1)[:, None]
    Zc = ((-1.0) ** i) * np.sqrt(2.0 / (n + 1)) * np.sin(i * k[None, :] * np.pi / (n + 1))
    rc = residuals(d, e, lam, Zc)
    ro = residuals(d, e, w, Z)
    ok = dk_comparable(lam, ro, rc)
    assert ok.sum() > 1000
    assert np.max(vec_diff_signfree(Z[:, ok], Zc[:, ok])) <= 1e-9
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1


@pytest.mark.parametrize("n", [3, 5, 7, 21, 101, 1001])
def test_zero_diagonal_closed_form(oracle_mod, n):
    """d = 0, e = 1: lambda_k = 2 cos(k pi / (n+1)) (the 1-2-1 spectrum shifted
    by -2); for odd n the middle eigenvalue is exactly 0 and its vector has a
    zero at every odd row -- an RQC that lands on a bracket end within
    rounding (reading 24's overshoot rule) must still converge to it."""
    d, e = np.zeros(n), np.ones(n - 1)
    w, Z = oracle_mod.stemr(d, e)
    lam = np.sort(2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    assert np.max(np.abs(w - lam)) <= 4 * n * EPS * tnorm1(d, e)
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1


@pytest.mark.parametrize("n", [64, 400, 1000])
def test_clement_closed_form(oracle_mod, n):
    d, e = W.clement(n)
    w, Z = oracle_mod.stemr(d, e)
    lam = 2.0 * np.arange(1, n + 1) - n - 1
    tn = tnorm1(d, e)
    assert np.max(np.abs(w - lam)) <= 4 * n * EPS * tn
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1


def test_interior_shift_strategy(oracle_mod):
    """Reading 30 (shift_strategy 1: an interior child shift for clusters of
    >= 2000 members) against the default 0 (end shifts only): on Clement n=4000 (one root cluster of ~3000 members,
    peeled from one end per level by end shifts) the eigenvalues still equal
    the closed form, the accuracy contract holds, and the tree is shallower
    than the end shifts' chain."""
    n = 4000
    d, e = W.clement(n)
    w0, Z0, st0 = oracle_mod.stemr(d, e, opts=oracle_mod.default_opts(shift_strategy=0), return_stats=True)
    w1, Z1, st1 = oracle_mod.stemr(d, e, return_stats=True)  # the default: interior first
    assert oracle_mod.default_opts().shift_strategy == 1
    lam = 2.0 * np.arange(1, n + 1) - n - 1
    tn = tnorm1(d, e)
    assert np.max(np.abs(w1 - lam)) <= 4 * n * EPS * tn
    res, orth = check_accuracy(d, e, w1, Z1)
    assert res <= 1 and orth <= 1
    assert st1["interior"] >= 1 and st0["interior"] == 0
    assert st1["max_depth"] < st0["max_depth"]


def test_clement_50000_subset_closed_form(oracle_mod):
    """configs[3] subset shape (first 40 of il..iu=1..5000): lambda_k = 2k-n-1."""
    n = 50000
    d, e = W.clement(n)
    w, Z = oracle_mod.stemr(d, e, il=1, iu=40)
    lam = 2.0 * np.arange(1, 41) - n - 1
    tn = tnorm1(d, e)
    assert np.max(np.abs(w - lam)) <= 4 * n * EPS * tn
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1


FAMILIES_SMALL = {
    "random_s0_64": lambda: W.random_uniform(64, 0),
    "random_s1_50": lambda: W.random_uniform(50, 1),
    "random_s2_33": lambda: W.random_uniform(33, 2),
    "wilkinson_21": lambda: W.wilkinson(21),
    "wilkinson_63": lambda: W.wilkinson(63),
    "one_two_one_64": lambda: W.one_two_one(64),
    "clement_64": lambda: W.clement(64),
    "glued_w21x3": lambda: W.glued_wilkinson(3),
    "tiny_2": lambda: (np.array([1.0, -2.0]), np.array([0.5])),
    "tiny_3": lambda: (np.array([0.0, 0.0, 0.0]), np.array([1.0, 1.0])),
}


@pytest.mark.parametrize("name", list(FAMILIES_SMALL))
def test_vs_jacobi_small(oracle_mod, name):
    """Brute-force dense Jacobi for n <= 64 (north_star (4))."""
    d, e = FAMILIES_SMALL[name]()
    n = len(d)
    w, Z = oracle_mod.stemr(d, e)
    wj, Vj = oracle_mod.jacobi(dense_T(d, e))
    tn = tnorm1(d, e)
    assert np.max(np.abs(w - wj)) <= 4 * n * EPS * tn
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1
    ok = dk_comparable(wj, residuals(d, e, w, Z), residuals(d, e, wj, Vj))
    if ok.any():
        assert np.max(vec_diff_signfree(Z[:, ok], Vj[:, ok])) <= 1e-9


@pytest.mark.parametrize("copies", [10, 40])
def test_glued_wilkinson_weyl(oracle_mod, copies):
    """configs[2] shape: |lambda_i - mu_ceil(i/copies)| <= 1e-8 (Weyl: the glue
    matrix has 2-norm 1e-8), mu = W21+ eigenvalues by Jacobi; exact trace and
    sum of squares identities."""
    d, e = W.glued_wilkinson(copies)
    n = len(d)
    w, Z = oracle_mod.stemr(d, e)
    db, eb = W.wilkinson(21)
    mu, _ = oracle_mod.jacobi(dense_T(db, eb))
    ref = np.repeat(mu, copies)
    assert np.max(np.abs(w - ref)) <= 1e-8 + 4 * n * EPS * tnorm1(d, e)
    tn = tnorm1(d, e)
    assert abs(w.sum() - d.sum()) <= n * 4 * n * EPS * tn
    assert abs((w ** 2).sum() - ((d ** 2).sum() + 2 * (e ** 2).sum())) <= n * 4 * n * EPS * tn * tn
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_invariants_and_lapack(oracle_mod, seed):
    """configs[1] shape at n=1500: residual, orthogonality, trace, sum of squares,
    Sturm placement with an independent numpy Sturm count, LAPACK stemr."""
    n = 1500
    d, e = W.random_uniform(n, seed)
    w, Z = oracle_mod.stemr(d, e)
    tn = tnorm1(d, e)
    tol = 4 * n * EPS * tn
    assert np.all(np.diff(w) >= 0)
    assert abs(w.sum() - d.sum()) <= n * tol
    assert abs((w ** 2).sum() - ((d ** 2).sum() + 2 * (e ** 2).sum())) <= n * tol * tn
    assert sturm_placement(d, e, w, np.arange(n), tol)
    wl, Vl = sl.eigh_tridiagonal(d, e, lapack_driver="stemr")
    assert np.max(np.abs(w - wl)) <= tol
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1
    ok = dk_comparable(wl, residuals(d, e, w, Z), residuals(d, e, wl, Vl))
    assert ok.sum() > n // 4
    assert np.max(vec_diff_signfree(Z[:, ok], Vl[:, ok])) <= 1e-9


def test_index_subset_consistent_with_all(oracle_mod):
    n = 800
    d, e = W.random_uniform(n, 4)
    wa, Za = oracle_mod.stemr(d, e)
    tn = tnorm1(d, e)
    for il, iu in [(1, 120), (300, 420), (701, 800), (17, 17)]:
        w, Z = oracle_mod.stemr(d, e, il=il, iu=iu)
        assert len(w) == iu - il + 1
        assert np.max(np.abs(w - wa[il - 1:iu])) <= 4 * n * EPS * tn
        res, orth = check_accuracy(d, e, w, Z)
        assert res <= 1 and orth <= 1
        ok = dk_comparable(wa[il - 1:iu], residuals(d, e, w, Z), residuals(d, e, wa[il - 1:iu], Za[:, il - 1:iu]))
        if ok.any():
            assert np.max(vec_diff_signfree(Z[:, ok], Za[:, il - 1:iu][:, ok])) <= 1e-9


def test_value_range(oracle_mod):
    n = 600
    d, e = W.random_uniform(n, 6)
    wa, _ = oracle_mod.stemr(d, e, vectors=False)
    vl, vu = -0.5, 0.25
    w, Z = oracle_mod.stemr(d, e, vl=vl, vu=vu)
    from helpers import sturm_numpy
    cnt = int(sturm_numpy(d, e, vu)[0] - sturm_numpy(d, e, vl)[0])
    assert len(w) == cnt
    assert np.all(w > vl - 1e-12) and np.all(w <= vu + 1e-12)
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1
    w0, Z0 = oracle_mod.stemr(d, e, vl=10.0, vu=11.0)
    assert len(w0) == 0


def test_values_only_matches(oracle_mod):
    n = 700
    d, e = W.random_uniform(n, 8)
    w1, _ = oracle_mod.stemr(d, e, vectors=False)
    w2, _ = oracle_mod.stemr(d, e)
    assert np.max(np.abs(w1 - w2)) <= 4 * n * EPS * tnorm1(d, e)
    wl = sl.eigvalsh_tridiagonal(d, e)
    assert np.max(np.abs(w1 - wl)) <= 4 * n * EPS * tnorm1(d, e)


def split_matrix():
    """Three irreducible blocks (exact zeros in e) with interleaved spectra."""
    d1, e1 = W.random_uniform(40, 11)
    d2, e2 = W.one_two_one(25)
    d3, e3 = W.wilkinson(21)
    d = np.concatenate([d1, d2 - 1.0, d3 * 0.2])
    e = np.concatenate([e1, [0.0], e2, [0.0], e3 * 0.2])
    return d, e


def test_multiblock_all_and_index(oracle_mod):
    d, e = split_matrix()
    n = len(d)
    assert len(oracle_mod.split(d, e)) == 4
    w, Z = oracle_mod.stemr(d, e)
    wj, Vj = oracle_mod.jacobi(dense_T(d, e))
    tn = tnorm1(d, e)
    assert np.max(np.abs(w - wj)) <= 4 * n * EPS * tn
    res, orth = check_accuracy(d, e, w, Z)
    assert res <= 1 and orth <= 1
    # rows outside a column's block are exactly zero
    nz = np.count_nonzero(Z, axis=0)
    assert np.all(nz <= 40)
    for il, iu in [(1, 30), (20, 60), (50, 86), (86, 86)]:
        wi, Zi = oracle_mod.stemr(d, e, il=il, iu=iu)
        assert len(wi) == iu - il + 1
        assert np.max(np.abs(wi - wj[il - 1:iu])) <= 4 * n * EPS * tn
        res, orth = check_accuracy(d, e, wi, Zi)
        assert res <= 1 and orth <= 1
    wv, Zv = oracle_mod.stemr(d, e, vl=-0.3, vu=0.4)
    ref = wj[(wj > -0.3) & (wj <= 0.4)]
    assert len(wv) == len(ref) and np.max(np.abs(wv - ref)) <= 4 * n * EPS * tn


def test_diagonal_and_tiny(oracle_mod):
    d = np.array([3.0, -1.0, 2.0, 2.0])
    w, Z = oracle_mod.stemr(d, np.zeros(3))
    assert list(w) == [-1.0, 2.0, 2.0, 3.0]
    assert np.array_equal(np.abs(Z.T @ Z), np.eye(4))
    w, Z = oracle_mod.stemr(np.array([7.5]), np.zeros(0))
    assert w[0] == 7.5 and Z[0, 0] == 1.0
    w, Z = oracle_mod.stemr(np.array([1.0, 1.0]), np.array([1.0]))
    assert np.allclose(w, [0.0, 2.0], atol=8 * EPS)


def test_argument_validation(oracle_mod):
    d, e = W.random_uniform(10, 0)
    assert oracle_mod.stemr_raw(0, d, e, 0, 0, 0, 0, 0) == -1
    bad = d.copy(); bad[3] = np.nan
    assert oracle_mod.stemr_raw(10, bad, e, 0, 0, 0, 0, 0) == -2
    bade = e.copy(); bade[0] = np.inf
    assert oracle_mod.stemr_raw(10, d, bade, 0, 0, 0, 0, 0) == -3
    assert oracle_mod.stemr_raw(10, d, e, 7, 0, 0, 0, 0) == -4
    assert oracle_mod.stemr_raw(10, d, e, 2, 1.0, 1.0, 0, 0) == -6
    assert oracle_mod.stemr_raw(10, d, e, 1, 0, 0, 0, 3) == -7
    assert oracle_mod.stemr_raw(10, d, e, 1, 0, 0, 4, 3) == -8
    assert oracle_mod.stemr_raw(10, d, e, 1, 0, 0, 4, 11) == -8
    assert oracle_mod.stemr_raw(10, d, e, 0, 0, 0, 0, 0, m_ptr_ok=False) == -9
    assert oracle_mod.stemr_raw(10, d, e, 0, 0, 0, 0, 0, w_ok=False) == -10
    assert oracle_mod.stemr_raw(10, d, e, 0, 0, 0, 0, 0, ldz=9) == -12
    assert oracle_mod.stemr_raw(10, d, e, 0, 0, 0, 0, 0) == 0


def test_deterministic(oracle_mod):
    d, e = W.glued_wilkinson(8)
    w1, Z1 = oracle_mod.stemr(d, e)
    w2, Z2 = oracle_mod.stemr(d, e)
    assert np.array_equal(w1, w2) and np.array_equal(Z1, Z2)


def test_stats_shape(oracle_mod):
    d, e = W.glued_wilkinson(20)
    w, Z, st = oracle_mod.stemr(d, e, return_stats=True)
    assert st["singletons"] == len(d)
    assert st["nodes"] >= 20 and st["max_depth"] >= 2   # degenerate copies need a tree
    assert sum(st["rqc_hist"]) == len(d)
