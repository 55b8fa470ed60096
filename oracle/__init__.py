"""Oracle loader -- TEST INFRASTRUCTURE ONLY.

ctypes binding of ``oracle/liboracle.so`` (plain sequential C MRRR, see
``mrrr_oracle.h``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this.
The product package ``paper_1205_2107_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "mrrr_oracle.c")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11", "-Wall",
          "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, IEEE division)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "mrrr_oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


class Opts(C.Structure):
    _fields_ = [("tol_relgap", C.c_double), ("rtol_class", C.c_double),
                ("max_depth", C.c_int), ("perturb_root", C.c_int),
                ("seed", C.c_uint64), ("rtol_vec", C.c_double), ("rqc_max", C.c_int),
                ("shift_strategy", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("negcount_sweeps", C.c_int64), ("negcount_resweeps", C.c_int64),
                ("child_sweeps", C.c_int64), ("twisted", C.c_int64),
                ("twisted_resweeps", C.c_int64), ("rqc_fallbacks", C.c_int64),
                ("nodes", C.c_int64), ("max_depth", C.c_int64),
                ("singletons", C.c_int64), ("root_retries", C.c_int64),
                ("tier", C.c_int64 * 4), ("rqc_hist", C.c_int64 * 12), ("interior", C.c_int64)]

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if not isinstance(v, int) else v
        return out


_lib = None
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.oracle_default_opts.argtypes = [C.POINTER(Opts)]
        L.oracle_stemr.argtypes = [C.c_int64, _dp, _dp, C.c_int, C.c_double, C.c_double,
                                   C.c_int64, C.c_int64, C.POINTER(Opts), _i64p, _dp, _dp,
                                   C.c_int64, C.POINTER(Stats)]
        L.oracle_stemr.restype = C.c_int
        L.oracle_norms.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, _dp]
        L.oracle_split.argtypes = [C.c_int64, _dp, _dp, C.c_double, _i64p]
        L.oracle_split.restype = C.c_int64
        L.oracle_root_rrr.argtypes = [C.c_int64, _dp, _dp, C.c_double, C.c_int, C.c_int,
                                      C.c_uint64, C.c_int64, _dp, _dp, _dp, _i64p]
        L.oracle_root_rrr.restype = C.c_int
        L.oracle_negcount.argtypes = [C.c_int64, _dp, _dp, C.c_double, C.c_double,
                                      C.POINTER(C.c_int)]
        L.oracle_negcount.restype = C.c_int64
        L.oracle_sturm_T.argtypes = [C.c_int64, _dp, _dp, C.c_double]
        L.oracle_sturm_T.restype = C.c_int64
        L.oracle_classify.argtypes = [C.c_int64, _dp, _dp, C.c_double, C.POINTER(C.c_int)]
        L.oracle_child_rrr.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp]
        L.oracle_child_rrr.restype = C.c_int
        L.oracle_twisted.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, C.c_double, C.c_double,
                                     _dp, _i64p, _dp, _i64p]
        L.oracle_twisted.restype = C.c_int
        L.oracle_jacobi.argtypes = [C.c_int64, _dp, _dp, _dp]
        L.oracle_jacobi.restype = C.c_int
        L.oracle_perturb_u.argtypes = [C.c_uint64, C.c_int64, C.c_int]
        L.oracle_perturb_u.restype = C.c_double
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().oracle_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle_stemr returned {code}")
        self.code = code


def stemr(d, e, *, il=None, iu=None, vl=None, vu=None, vectors=True, opts=None,
          return_stats=False):
    """Oracle MRRR: (w, Z) with Z[:, j] the unit eigenvector of w[j]."""
    d = _f64(d)
    n = d.shape[0]
    e = _f64(e) if n > 1 else np.zeros(1)
    if il is not None:
        rng, a, b = 1, int(il), int(iu)
        kmax = max(0, b - a + 1)
    elif vl is not None:
        rng, a, b = 2, 0, 0
        kmax = n
    else:
        rng, a, b = 0, 0, 0
        kmax = n
    w = np.zeros(max(kmax, 1))
    Zf = np.zeros((max(kmax, 1), n)) if vectors else None  # column j = row j (C order)
    m = C.c_int64(0)
    st = Stats()
    o = opts if opts is not None else default_opts()
    rc = lib().oracle_stemr(n, _p(d), _p(e), rng, float(vl or 0.0), float(vu or 0.0), a, b,
                            C.byref(o), C.byref(m), _p(w),
                            _p(Zf) if vectors else C.cast(None, _dp), n, C.byref(st))
    if rc != 0:
        raise OracleError(rc)
    k = m.value
    w = w[:k].copy()
    Z = Zf[:k].T.copy() if vectors else None
    if return_stats:
        return w, Z, st.as_dict()
    return w, Z


def stemr_raw(n, d, e, rng, vl, vu, il, iu, m_ptr_ok=True, w_ok=True, ldz=None, vectors=True):
    """Direct call for argument-validation tests; returns the C return code."""
    d = _f64(d)
    e = _f64(e)
    w = np.zeros(max(n, 1))
    Zf = np.zeros((max(n, 1), max(n, 1)))
    m = C.c_int64(0)
    rc = lib().oracle_stemr(n, _p(d), _p(e), rng, vl, vu, il, iu, None,
                            C.byref(m) if m_ptr_ok else C.cast(None, _i64p),
                            _p(w) if w_ok else C.cast(None, _dp),
                            _p(Zf) if vectors else C.cast(None, _dp),
                            ldz if ldz is not None else max(n, 1), None)
    return rc


def norms(d, e):
    d, e = _f64(d), _f64(e)
    t, g0, g1 = C.c_double(), C.c_double(), C.c_double()
    lib().oracle_norms(d.shape[0], _p(d), _p(e), C.byref(t), C.byref(g0), C.byref(g1))
    return t.value, g0.value, g1.value


def split(d, e):
    d, e = _f64(d), _f64(e)
    n = d.shape[0]
    t, _, _ = norms(d, e)
    bs = np.zeros(n + 1, dtype=np.int64)
    nb = lib().oracle_split(n, _p(d), _p(e), t, bs.ctypes.data_as(_i64p))
    return bs[: nb + 1].copy()


def root_rrr(d, e, side=1, perturb=0, seed=0):
    d, e = _f64(d), _f64(e)
    n = d.shape[0]
    t, _, _ = norms(d, e)
    D = np.zeros(n)
    L = np.zeros(max(n - 1, 1))
    s = C.c_double()
    r = C.c_int64(0)
    rc = lib().oracle_root_rrr(n, _p(d), _p(e), t, side, perturb, seed, 0, _p(D), _p(L),
                               C.byref(s), C.byref(r))
    if rc:
        raise OracleError(rc)
    return D, L[: n - 1].copy(), s.value


def negcount(D, L, mu, LLD=None, return_resweep=False):
    """O6 count N(mu) of L D L^T; LLD may be given directly (then L is unused).
    With return_resweep, also whether the NaN-safe re-sweep ran (a zero pivot)."""
    D = _f64(D)
    if LLD is None:
        L = _f64(L)
        LLD = L * L * D[:-1] if len(L) else np.zeros(1)
    LLD = _f64(LLD) if len(LLD) else np.zeros(1)
    piv = np.finfo(float).tiny * max(1.0, float(np.max(np.abs(LLD))))
    rs = C.c_int(0)
    c = lib().oracle_negcount(D.shape[0], _p(D), _p(LLD), float(mu), piv, C.byref(rs))
    return (c, bool(rs.value)) if return_resweep else c


def sturm_T(d, e, x):
    d, e = _f64(d), _f64(e)
    return lib().oracle_sturm_T(d.shape[0], _p(d), _p(e), float(x))


def classify(lo, hi, tol=1e-3):
    lo, hi = _f64(lo), _f64(hi)
    k = lo.shape[0]
    out = (C.c_int * max(k - 1, 1))()
    lib().oracle_classify(k, _p(lo), _p(hi), tol, out)
    return [int(out[i]) for i in range(k - 1)]


def child_rrr(D, L, sigma):
    D, L = _f64(D), _f64(L)
    n = D.shape[0]
    LD = _f64(L * D[:-1])
    Dp = np.zeros(n)
    Lp = np.zeros(max(n - 1, 1))
    g = C.c_double()
    rc = lib().oracle_child_rrr(n, _p(D), _p(L), _p(LD), float(sigma), _p(Dp), _p(Lp),
                                C.byref(g))
    return rc, Dp, Lp[: n - 1].copy(), g.value


def twisted(D, L, lam):
    D, L = _f64(D), _f64(L)
    n = D.shape[0]
    LD = _f64(L * D[:-1])
    LLD = _f64(L * LD)
    piv = np.finfo(float).tiny * max(1.0, float(np.max(np.abs(LLD))))
    z = np.zeros(n)
    r = C.c_int64()
    g = C.c_double()
    nc = C.c_int64()
    lib().oracle_twisted(n, _p(D), _p(L), _p(LD), _p(LLD), float(lam), piv, _p(z),
                         C.byref(r), C.byref(g), C.byref(nc))
    return z, r.value, g.value, nc.value


def jacobi(A):
    A = _f64(A)
    n = A.shape[0]
    w = np.zeros(n)
    V = np.zeros((n, n))
    rc = lib().oracle_jacobi(n, _p(A), _p(w), _p(V))
    if rc:
        raise OracleError(rc)
    return w, V


def perturb_u(seed, grow, tag):
    return lib().oracle_perturb_u(seed, grow, tag)
