"""Test-side metrics.  Independent of both the oracle's and the CUDA path's
arithmetic (plain numpy written from the definitions in BASELINE.json /
PAPER.md Eq. (Tresnorm), (Torthogo), L832-843)."""
from __future__ import annotations

import numpy as np

EPS = np.finfo(np.float64).eps


def tnorm1(d, e):
    """||T||_1 = max_i |e_{i-1}| + |d_i| + |e_i|."""
    d = np.asarray(d, float)
    e = np.asarray(e, float)
    r = np.abs(d).copy()
    if len(e):
        r[:-1] += np.abs(e)
        r[1:] += np.abs(e)
    return float(r.max())


def tmatvec(d, e, Z):
    """T @ Z for T = tridiag(e, d, e), Z n x k."""
    TZ = d[:, None] * Z
    if len(e):
        TZ[1:] += e[:, None] * Z[:-1]
        TZ[:-1] += e[:, None] * Z[1:]
    return TZ


def residuals(d, e, w, Z):
    """||T z_j - w_j z_j||_2 per column."""
    return np.linalg.norm(tmatvec(d, e, Z) - Z * w[None, :], axis=0)


def orthogonality(Z):
    k = Z.shape[1]
    O = Z.T @ Z - np.eye(k)
    return float(np.max(np.abs(O))) if k else 0.0


def sturm_numpy(d, e, xs):
    """#eigenvalues of T below each x (classic Sturm sequence, vectorised over x,
    zero pivot treated as a tiny negative).  Independent of the oracle."""
    xs = np.atleast_1d(np.asarray(xs, float))
    tiny = np.finfo(float).tiny
    piv = tiny * max(1.0, float(np.max(e * e)) if len(e) else 1.0)
    q = d[0] - xs
    q = np.where(np.abs(q) < piv, -piv, q)
    c = (q < 0).astype(np.int64)
    for i in range(1, len(d)):
        q = (d[i] - xs) - (e[i - 1] * e[i - 1]) / q
        q = np.where(np.abs(q) < piv, -piv, q)
        c += q < 0
    return c


NFLOOR = 1000


def check_accuracy(d, e, w, Z, *, nfloor=NFLOOR):
    """BASELINE.json tolerances: residual/||T||_1 <= 10 n eps, orthogonality
    <= 10 n eps, with n floored at 1/tol = 1000 (reading 26: the
    paper's error-angle bound |sin angle| <= O(n eps / relgap) (Eq. errorangle,
    P:L1086-1090) with relgap just above tol = 1e-3 allows eps/tol = 1000 eps
    at any n; LAPACK dstemr itself reaches 4.4x of 10 n eps at Wilkinson
    n=21.  Every BASELINE config has n >= 2000, where the floor is inactive).  Returns the normalised metrics
    (<= 1 passes)."""
    n = max(len(d), nfloor)
    tn = tnorm1(d, e)
    res = float(np.max(residuals(d, e, w, Z))) / tn / (10 * n * EPS) if Z.shape[1] else 0.0
    orth = orthogonality(Z) / (10 * n * EPS)
    return res, orth


def sturm_placement(d, e, w, idx0, delta):
    """N_T(w_j - delta) <= j-1 < N_T(w_j + delta) for global (0-based) index j."""
    lo = sturm_numpy(d, e, w - delta)
    hi = sturm_numpy(d, e, w + delta)
    j = np.asarray(idx0)
    return np.all(lo <= j) and np.all(j < hi)


def dk_comparable(w_ref, r_a, r_b, idx=None):
    """Davis-Kahan rule (SURVEY §8(c) reading 18): compare vector j iff
    (r_a + r_b) / gap_j <= 1e-10, gap from the reference eigenvalues."""
    w = np.asarray(w_ref, float)
    k = len(w)
    gap = np.full(k, np.inf)
    if k > 1:
        dw = np.diff(w)
        gap[:-1] = np.minimum(gap[:-1], dw)
        gap[1:] = np.minimum(gap[1:], dw)
    with np.errstate(divide="ignore", invalid="ignore"):
        ok = (r_a + r_b) / gap <= 1e-10
    return ok


def vec_diff_signfree(za, zb):
    """min(||za - zb||_inf, ||za + zb||_inf) per column (reading 12)."""
    a = np.max(np.abs(za - zb), axis=0)
    b = np.max(np.abs(za + zb), axis=0)
    return np.minimum(a, b)


def subspace_runs(w_ref, r_a, r_b, ok, full_range=True):
    """The eigenpairs that are NOT individually comparable (dk_comparable
    false: inside clusters or degenerate groups, where any orthonormal basis
    of the invariant subspace is correct) grouped into maximal runs of
    consecutive indices.  A run's invariant subspace is unique when it is
    well separated from the other eigenvalues: by Davis-Kahan, sin(theta)
    between the subspace a basis spans and the exact one is at most
    ||R||_F / gap_out, so two bases with (||R_a||_F + ||R_b||_F) / gap_out <=
    1e-10 must span the same subspace to that accuracy.  Returns the
    half-open index ranges (a, b) of such runs.  For an index or value
    subset (full_range=False) runs touching the ends are skipped: their
    nearest outside eigenvalue is not in the list."""
    w = np.asarray(w_ref, float)
    k = len(w)
    out = []
    i = 0
    while i < k:
        if ok[i]:
            i += 1
            continue
        j = i
        while j < k and not ok[j]:
            j += 1
        a, b = i, j
        i = j
        if not full_range and (a == 0 or b == k):
            continue
        gl = w[a] - w[a - 1] if a > 0 else np.inf
        gr = w[b] - w[b - 1] if b < k else np.inf
        gap = min(gl, gr)
        R = np.sqrt(np.sum(r_a[a:b] ** 2)) + np.sqrt(np.sum(r_b[a:b] ** 2))
        if gap == np.inf or R / gap <= 1e-10:
            out.append((a, b))
    return out


def subspace_diff(Za, Zb):
    """max over the columns of Za of ||z - Zb Zb^T z||_2: how far Za's columns
    lie from the span of Zb's (orthonormal) columns."""
    P = Za - Zb @ (Zb.T @ Za)
    return float(np.max(np.linalg.norm(P, axis=0))) if Za.shape[1] else 0.0
