"""Zero-diagonal tridiagonals (exact eigenvalue 0 for odd n, a zero middle
component): residual per root refinement width (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1205_2107_b200 as P  # noqa: E402

for n in (3, 5, 7, 9, 11, 21, 101, 1001):
    out = []
    for m in ("1", "2", "4"):
        os.environ["MRRR_RW_ROOT_M"] = m
        d = np.zeros(n); e = np.ones(n - 1)
        w, Z = P.stemr(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda"))
        w = w.cpu().numpy(); Z = Z.cpu().numpy()
        T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        res = np.max(np.linalg.norm(T @ Z - Z * w, axis=0)) / (3 * n * 2.0 ** -52 * 10)
        st = P.last_stats()
        out.append(f"M{m}: res/bound {res:.3g} rqc {st['rqc_iters']} fb {st['rqc_fallbacks']}")
    print(n, " | ".join(out))
