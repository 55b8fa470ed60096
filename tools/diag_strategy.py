"""Diagnostics (test tooling): the child-shift strategies (mrrr_opts_t
shift_strategy 0 = cluster ends, 1 = interior first, reading 30)
on BASELINE configs: levels, nodes, time (CUDA events, best of 3), residual
and orthogonality on the GPU (sampled 4096-column blocks for n > 30000).
usage: python tools/diag_strategy.py config [config ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_2107_b200 as P  # noqa: E402
from paper_1205_2107_b200 import workloads as W  # noqa: E402

EPS = 2.0 ** -52
for name in sys.argv[1:]:
    d, e, rng = W.make(name)
    n = len(d)
    kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
    dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
    r = np.abs(d).copy(); r[:-1] += np.abs(e); r[1:] += np.abs(e)
    tn = float(r.max())
    P.trim_workspace()
    k0 = n if rng is None else rng[1] - rng[0] + 1
    wbuf = torch.empty(k0, dtype=torch.float64, device="cuda")
    Zbuf = torch.empty((k0, n), dtype=torch.float64, device="cuda")
    for strat in [int(x) for x in os.environ.get("STRATS", "0,1").split(",")]:
        o = P.default_opts(shift_strategy=strat)
        best = None
        for it in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            w, Z = P.stemr(dt, et, opts=o, w=wbuf, Z=Zbuf, **kw)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        st = P.last_stats()
        P.trim_workspace()  # the metrics below need the memory
        k = w.shape[0]
        B = 4096
        res = 0.0
        orth = 0.0
        blocks = list(range(0, k, B))
        if n > 30000 and not os.environ.get("FULL"):
            blocks = blocks[::4]
        worst = (0.0, -1, -1)
        for a0 in blocks:
            Zb = Z[:, a0:a0 + B]
            TZ = dt[:, None] * Zb
            TZ[1:] += et[:, None] * Zb[:-1]
            TZ[:-1] += et[:, None] * Zb[1:]
            R = TZ - Zb * w[None, a0:a0 + B]
            res = max(res, float(torch.linalg.vector_norm(R, dim=0).max()))
            G = Z.T @ Zb
            idx = torch.arange(Zb.shape[1], device="cuda")
            G[a0 + idx, idx] -= 1.0
            Ga = G.abs()
            v, flat = Ga.flatten().max(0)
            if float(v) > worst[0]:
                worst = (float(v), int(flat) // Ga.shape[1], a0 + int(flat) % Ga.shape[1])
            orth = max(orth, float(v))
            del TZ, R, G
        print(json.dumps({"config": name, "shift_strategy": strat, "int_wg": os.environ.get("MRRR_INT_WG", "64"),
                          "ms": round(best, 2),
                          "levels": st["levels"], "nodes": st["nodes"],
                          "res": res / tn / (10 * n * EPS), "orth": orth / (10 * n * EPS),
                          "worst_pair": [worst[1], worst[2], float(w[worst[1]]), float(w[worst[2]])] if worst[1] >= 0 else None}),
              flush=True)
        del w, Z, Zb
        torch.cuda.empty_cache()
