"""Seeded synthetic tridiagonal workloads (shared by tests, bench and smoke).

This module holds NO arithmetic of the method: it only generates the inputs
``(d, e)`` of ``T = tridiag(e, d, e)`` for the BASELINE.json configs.  Both the
oracle tests and the CUDA path consume the same arrays.

Families:
  * ``one_two_one(n)``      d_i = 2, e_i = 1           (config 1)
  * ``random_uniform(n,s)`` d, e iid U(-1,1), numpy default_rng(seed); d drawn
                            first, then e                  (configs 2 and 5)
  * ``glued_wilkinson(k)``  k copies of W21+ (d = |i-10|, inner e = 1) glued by
                            e = 1e-8                      (config 3)
  * ``clement(n)``          d = 0, e_i = sqrt(i (n-i))     (config 4)
  * ``wilkinson(n)``        d = (m, ..., 1, 0, 1, ..., m), e = 1, m=(n-1)/2
                            
"""
from __future__ import annotations

import numpy as np


def one_two_one(n: int):
    return np.full(n, 2.0), np.ones(max(n - 1, 0))


def random_uniform(n: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    d = rng.uniform(-1.0, 1.0, n)
    e = rng.uniform(-1.0, 1.0, max(n - 1, 0))
    return d, e


def wilkinson(n: int):
    m = (n - 1) // 2
    d = np.abs(np.arange(n, dtype=np.float64) - m)
    return d, np.ones(max(n - 1, 0))


def glued_wilkinson(copies: int, block: int = 21, glue: float = 1e-8):
    db, eb = wilkinson(block)
    d = np.tile(db, copies)
    e = np.ones(copies * block - 1)
    e[block - 1::block] = glue
    return d, e


def clement(n: int):
    i = np.arange(1, n, dtype=np.int64)
    return np.zeros(n), np.sqrt((i * (n - i)).astype(np.float64))


# BASELINE.json configs (name -> (builder, kwargs, range)); range is None for
# all pairs or (il, iu) 1-based inclusive.
CONFIGS = {
    "one_two_one_2000": (one_two_one, {"n": 2000}, None),
    "random_20000": (random_uniform, {"n": 20000, "seed": 0}, None),
    "glued_wilkinson_21000": (glued_wilkinson, {"copies": 1000}, None),
    "clement_50000_subset": (clement, {"n": 50000}, (1, 5000)),
    "clement_50000": (clement, {"n": 50000}, None),
    "random_100000": (random_uniform, {"n": 100000, "seed": 0}, None),
}


def make(name: str):
    fn, kw, rng = CONFIGS[name]
    d, e = fn(**kw)
    return d, e, rng
