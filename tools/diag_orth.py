"""Diagnostics (test tooling): run a config, report residual/orthogonality and
the worst orthogonality pair with its tree data (MRRR_DEBUG task dump)."""
import os, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_1205_2107_b200 as P
from paper_1205_2107_b200 import workloads as W
from helpers import tnorm1, EPS

name = sys.argv[1]
d, e, rng = W.make(name)
n = len(d)
kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
for it in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    w, Z = P.stemr(dt, et, **kw)
    torch.cuda.synchronize(); t1 = time.time()
    st = P.last_stats()
    print(f"{name} run {it}: wall {1e3*(t1-t0):.1f} ms stats {st}", flush=True)
k = w.shape[0]
best = (0.0, -1, -1)
B = 4096
for a in range(0, k, B):
    G = Z.T @ Z[:, a:a + B]
    idx = torch.arange(G.shape[1], device="cuda")
    G[a + idx, idx] -= 1.0
    G = G.abs()
    v, flat = G.flatten().max(0)
    if float(v) > best[0]:
        i, j = divmod(int(flat), G.shape[1])
        best = (float(v), i, a + j)
orth, i, j = best
print(f"orth {orth:.3e} = {orth/(10*n*EPS):.3f} x tol at pair ({i},{j}) w_i={float(w[i]):.17g} w_j={float(w[j]):.17g}")
wn = w.cpu().numpy()
for q in sorted({i, j}):
    lo, hi = max(q - 3, 0), min(q + 4, k)
    print("  neighbourhood", q, [f"{x:.17g}" for x in wn[lo:hi]])
# column-wise worst orthogonality counts
cnt = 0
tol = 10 * n * EPS
for a in range(0, k, B):
    G = Z.T @ Z[:, a:a + B]
    idx = torch.arange(G.shape[1], device="cuda")
    G[a + idx, idx] -= 1.0
    cnt += int((G.abs() > tol).sum())
print("entries over tol:", cnt)
