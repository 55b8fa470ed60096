"""Pins for the oracle's step functions (CPU only).  Each pin is something the
paper, SPEC's worked examples or plain linear algebra fixes -- never the oracle
re-called on itself (task ③)."""
import json
import os

import numpy as np
import pytest

from helpers import EPS
from paper_1205_2107_b200 import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def dense_T(d, e):
    return np.diag(d) + np.diag(e, 1) + np.diag(e, -1)


def dense_LDLT(D, L):
    n = len(D)
    Lm = np.eye(n) + np.diag(L, -1)
    return Lm @ np.diag(D) @ Lm.T


def test_sturm_T_spec_example(oracle_mod):
    g = GOLD["sturm_count"][0]
    d, e = W.one_two_one(g["n"])
    assert oracle_mod.sturm_T(d, e, g["mu"]) == g["count"]


def test_negcount_spec_example_shifted(oracle_mod):
    """S:L250-252 in shifted coordinates of the root RRR, both sides."""
    d, e = W.one_two_one(4)
    for side in (1, -1):
        D, L, s = oracle_mod.root_rrr(d, e, side=side)
        assert oracle_mod.negcount(D, L, 2.0 - s) == 2
        ev = GOLD["sturm_count"][1]["eigenvalues_approx"]
        for k, lam in enumerate(ev):
            assert oracle_mod.negcount(D, L, lam - s - 1e-5) == k
            assert oracle_mod.negcount(D, L, lam - s + 1e-5) == k + 1


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("perturb", [0, 1])
def test_negcount_vs_dense_counts(oracle_mod, seed, perturb):
    """O6 count == #eigenvalues of the dense L D L^T below mu (numpy eigvalsh)."""
    d, e = W.random_uniform(60, seed)
    D, L, s = oracle_mod.root_rrr(d, e, side=1, perturb=perturb, seed=7)
    ev = np.linalg.eigvalsh(dense_LDLT(D, L))
    rng = np.random.default_rng(seed)
    mus = np.concatenate([rng.uniform(ev[0] - 0.1, ev[-1] + 0.1, 300), ev * (1 + 1e-7), ev * (1 - 1e-7)])
    for mu in mus:
        assert oracle_mod.negcount(D, L, mu) == int(np.sum(ev < mu))


def test_negcount_zero_pivots_clement(oracle_mod):
    """Exact zero pivots (Clement at the T-origin: odd leading minors of a zero
    diagonal tridiagonal vanish).  The count must equal the true count n/2."""
    for n in (10, 400):
        d, e = W.clement(n)
        D, L, s = oracle_mod.root_rrr(d, e, side=1, perturb=0)
        assert oracle_mod.negcount(D, L, -s) == n // 2


@pytest.mark.parametrize("fam", ["one_two_one", "random", "clement", "wilkinson"])
@pytest.mark.parametrize("side", [1, -1])
def test_root_rrr_reconstruction(oracle_mod, fam, side):
    """|L D L^T + sigma I - T| <= 8 eps (|T| + |sigma|) elementwise;
    definite (all pivots of one sign); sigma outside the Gershgorin interval."""
    d, e = {"one_two_one": W.one_two_one(50), "random": W.random_uniform(50, 3),
            "clement": W.clement(50), "wilkinson": W.wilkinson(51)}[fam]
    D, L, s = oracle_mod.root_rrr(d, e, side=side, perturb=0)
    T = dense_T(d, e)
    R = dense_LDLT(D, L) + s * np.eye(len(d))
    assert np.all(np.abs(R - T) <= 8 * EPS * (np.abs(T) + abs(s)) + 1e-300)
    assert np.all(D > 0) if side > 0 else np.all(D < 0)
    tn, gl, gu = oracle_mod.norms(d, e)
    assert (s < gl) if side > 0 else (s > gu)


def test_root_perturbation_is_relative_4eps(oracle_mod):
    d, e = W.random_uniform(200, 0)
    D0, L0, s0 = oracle_mod.root_rrr(d, e, side=1, perturb=0)
    D1, L1, s1 = oracle_mod.root_rrr(d, e, side=1, perturb=1, seed=123)
    assert s0 == s1
    rd = np.abs(D1 / D0 - 1)
    rl = np.abs(L1 / L0 - 1)
    assert rd.max() <= 4.5 * EPS and rl.max() <= 4.5 * EPS
    assert np.count_nonzero(rd) > 150  # it does perturb


def test_perturb_generator_published_vectors(oracle_mod):
    """oracle_perturb_u(seed, g, tag) = u(sm(seed ^ sm(2g + tag))) with sm the
    splitmix64 output function and u(x) = (x >> 11) 2^-52 - 1 (DESIGN.md
    reading 3) is pinned to the generator's PUBLISHED outputs
    (tests/golden/splitmix64.json): sm(s) is the first output of splitmix64
    started at state s, so choosing the seed to cancel the inner value makes
    the outer call reproduce a published output.  A wrong constant, shift or
    composition fails here."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "splitmix64.json")))
    A = int(g["state0_first_three_outputs_hex"][0], 16)      # sm(0)
    C = int(g["seed1234567_first_three_outputs"][0])         # sm(1234567)

    def u(x):
        return float(x >> 11) * 2.0 ** -52 - 1.0
    # inner sm(0) = A: seed A ^ s gives the outer sm(s)
    assert oracle_mod.perturb_u(A, 0, 0) == u(A)
    assert oracle_mod.perturb_u(A ^ 1234567, 0, 0) == u(C)
    # inner sm(2 * 617283 + 1) = sm(1234567) = C
    assert oracle_mod.perturb_u(C, 617283, 1) == u(A)
    assert oracle_mod.perturb_u(C ^ 1234567, 617283, 1) == u(C)


def test_perturb_generator(oracle_mod):
    u = np.array([oracle_mod.perturb_u(99, i, t) for i in range(4000) for t in (0, 1)])
    assert np.all(u >= -1) and np.all(u < 1)
    assert abs(u.mean()) < 0.05 and 0.3 < u.std() < 0.7
    assert oracle_mod.perturb_u(99, 5, 0) == oracle_mod.perturb_u(99, 5, 0)
    assert oracle_mod.perturb_u(99, 5, 0) != oracle_mod.perturb_u(99, 5, 1)
    assert oracle_mod.perturb_u(99, 5, 0) != oracle_mod.perturb_u(98, 5, 0)


@pytest.mark.parametrize("case", GOLD["classify"], ids=lambda c: c["cite"])
def test_classify_spec_examples(oracle_mod, case):
    v = np.array(case["values"])
    bd = oracle_mod.classify(v, v, case["tol"])
    runs, s = [], 0
    for j in range(len(v)):
        if j == len(v) - 1 or bd[j]:
            runs.append([s + 1, j + 1])
            s = j + 1
    assert runs == case["runs"]


def test_classify_strict_and_conservative(oracle_mod):
    # gap exactly tol*max -> not a boundary (strict >, reading 6)
    assert oracle_mod.classify(np.array([1.0, 1.5]), np.array([1.0, 1.5]), 1.0 / 3.0) == [0]
    # the conservative gap uses lo_{j+1} - hi_j
    lo = np.array([1.0, 1.0025])
    hi = np.array([1.002, 1.003])
    assert oracle_mod.classify(lo, hi, 1e-3) == [0]
    assert oracle_mod.classify(lo, np.array([1.0, 1.003]), 1e-3) == [1]


@pytest.mark.parametrize("case", GOLD["split"], ids=lambda c: c["cite"])
def test_split_spec_examples(oracle_mod, case):
    bs = oracle_mod.split(np.array(case["d"]), np.array(case["e"]))
    assert list(bs) == case["bstart"]


def test_split_diagonal_eigenpairs(oracle_mod):
    case = GOLD["split"][0]
    w, Z = oracle_mod.stemr(np.array(case["d"]), np.array(case["e"]))
    for k, (lam, i) in enumerate(case["eigenpairs"]):
        assert w[k] == lam
        zz = np.zeros(3)
        zz[i] = 1
        assert np.array_equal(np.abs(Z[:, k]), zz)


def test_child_rrr_reconstruction(oracle_mod):
    """child reconstructs parent - sigma I elementwise (mixed stability)."""
    d, e = W.random_uniform(80, 5)
    D, L, s = oracle_mod.root_rrr(d, e, side=1, perturb=0)
    P = dense_LDLT(D, L)
    for sigma in (0.0, 0.37, 1.9, 2.5):
        rc, Dp, Lp, g = oracle_mod.child_rrr(D, L, sigma)
        assert rc == 0
        C = dense_LDLT(Dp, Lp)
        ref = P - sigma * np.eye(80)
        scale = np.abs(dense_LDLT(np.abs(D), np.abs(L))) + np.abs(dense_LDLT(np.abs(Dp), np.abs(Lp))) + abs(sigma)
        assert np.all(np.abs(C - ref) <= 16 * EPS * scale)
        assert g == np.max(np.abs(Dp))
    rc, Dp, Lp, g = oracle_mod.child_rrr(D, L, 0.0)
    assert np.array_equal(Dp, D) and np.allclose(Lp, L, rtol=2 * EPS, atol=0)


def test_child_rrr_diagonal_parent(oracle_mod):
    """decoupled parent (L = 0): D+ = D - sigma, L+ = 0."""
    D = np.array([1.0, 2.0, 3.0, 5.0])
    L = np.zeros(3)
    rc, Dp, Lp, g = oracle_mod.child_rrr(D, L, 0.5)
    assert np.array_equal(Dp, D - 0.5) and np.array_equal(Lp, np.zeros(3))


@pytest.mark.parametrize("seed", [0, 1])
def test_twisted_vs_dense_inverse(oracle_mod, seed):
    """O10 steps 1-4: gamma_r = 1/[(LDL^T - lam I)^-1]_rr, r = argmin |gamma|,
    (LDL^T - lam I) z = gamma_r e_r with z_r = 1, twisted negcount = dense count."""
    d, e = W.random_uniform(60, seed)
    D, L, s = oracle_mod.root_rrr(d, e, side=1, perturb=0)
    A = dense_LDLT(D, L)
    ev = np.linalg.eigvalsh(A)
    for j in (0, 7, 31, 59):
        lam = ev[j] * (1 + 1e-6)
        z, r, g, nc = oracle_mod.twisted(D, L, lam)
        M = A - lam * np.eye(60)
        Minv = np.linalg.inv(M)
        gam = 1.0 / np.diag(Minv)
        assert r == int(np.argmin(np.abs(gam)))
        assert abs(g - gam[r]) <= 1e-6 * abs(gam[r])
        assert z[r] == 1.0
        res = M @ z
        res[r] -= g
        assert np.max(np.abs(res)) <= 1e-12 * np.max(np.abs(z)) * np.max(np.abs(A))
        assert nc == int(np.sum(ev < lam))


def test_twisted_endpoints(oracle_mod):
    """gamma_1 = P_1 and gamma_n = D+_n: a vector for the extreme twist."""
    d, e = W.random_uniform(30, 9)
    D, L, s = oracle_mod.root_rrr(d, e, side=1, perturb=0)
    A = dense_LDLT(D, L)
    ev = np.linalg.eigvalsh(A)
    z, r, g, nc = oracle_mod.twisted(D, L, ev[0] * (1 + 1e-3))
    M = A - ev[0] * (1 + 1e-3) * np.eye(30)
    assert abs(g - 1 / np.linalg.inv(M)[r, r]) <= 1e-9 * abs(g)


def test_spec_eigenvector_121_n3(oracle_mod):
    g = GOLD["eigenvector"][0]
    d, e = W.one_two_one(3)
    w, Z = oracle_mod.stemr(d, e)
    j = int(np.argmin(np.abs(w - g["eigenvalue"])))
    ref = np.array(g["vector_times_sqrt2"]) / np.sqrt(2)
    assert min(np.max(np.abs(Z[:, j] - ref)), np.max(np.abs(Z[:, j] + ref))) <= 10 * 3 * EPS


def test_wilkinson_generator_spec():
    g = GOLD["wilkinson"][0]
    d, e = W.wilkinson(g["n"])
    assert list(d) == g["d"] and len(e) == g["n"] - 1 and np.all(e == g["e_all"])


# ---- Jacobi (the brute-force oracle for n <= 64) pinned to closed forms ----

def test_jacobi_2x2_spec(oracle_mod):
    g = GOLD["jacobi"][0]
    w, V = oracle_mod.jacobi(np.array(g["A"]))
    assert np.allclose(w, g["w"], atol=4 * EPS)
    ref = np.array(g["V_times_sqrt2"]) / np.sqrt(2)
    for j in range(2):
        assert min(np.max(np.abs(V[:, j] - ref[:, j])), np.max(np.abs(V[:, j] + ref[:, j]))) <= 4 * EPS


def test_jacobi_diagonal_exact(oracle_mod):
    A = np.diag([3.0, -1.0, 2.0, 0.5])
    w, V = oracle_mod.jacobi(A)
    assert list(w) == [-1.0, 0.5, 2.0, 3.0]
    assert np.array_equal(np.abs(V), np.eye(4)[:, [1, 3, 2, 0]])


def test_jacobi_121_analytic(oracle_mod):
    n = 8
    d, e = W.one_two_one(n)
    w, V = oracle_mod.jacobi(dense_T(d, e))
    k = np.arange(1, n + 1)
    assert np.max(np.abs(w - (2 - 2 * np.cos(k * np.pi / (n + 1))))) <= 10 * n * EPS


@pytest.mark.parametrize("n", [5, 17, 64])
def test_jacobi_random_symmetric_invariants(oracle_mod, n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    A = A + A.T
    w, V = oracle_mod.jacobi(A)
    nrm = np.linalg.norm(A)
    assert abs(w.sum() - np.trace(A)) <= 50 * n * EPS * nrm
    assert abs((w ** 2).sum() - nrm ** 2) <= 100 * n * EPS * nrm ** 2
    assert np.max(np.abs(A @ V - V * w)) <= 50 * n * EPS * nrm
    assert np.max(np.abs(V.T @ V - np.eye(n))) <= 50 * n * EPS
    assert np.all(np.diff(w) >= 0)
