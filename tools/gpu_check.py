"""Ad-hoc GPU check: run the CUDA solver on several families, compare with the
oracle and print normalised metrics (<= 1 passes).  Test tooling only."""
import sys, time, traceback
import numpy as np
import torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle
from helpers import check_accuracy, tnorm1, residuals, dk_comparable, vec_diff_signfree, EPS
import paper_1205_2107_b200 as P
from paper_1205_2107_b200 import workloads as W

cases = [
    ("121_10", W.one_two_one(10), {}),
    ("rand_50", W.random_uniform(50, 0), {}),
    ("rand_400", W.random_uniform(400, 0), {}),
    ("wilk_201", W.wilkinson(201), {}),
    ("glued_10", W.glued_wilkinson(10), {}),
    ("clem_400", W.clement(400), {}),
    ("121_2000", W.one_two_one(2000), {}),
    ("rand_3000", W.random_uniform(3000, 0), {}),
    ("glued_200", W.glued_wilkinson(200), {}),
    ("rand_1000_idx", W.random_uniform(1000, 1), {"il": 101, "iu": 300}),
    ("clem_3000_idx", W.clement(3000), {"il": 1, "iu": 300}),
]
only = sys.argv[1:]
for name, (d, e), kw in cases:
    if only and name not in only:
        continue
    try:
        n = len(d)
        dt = torch.tensor(d, device='cuda'); et = torch.tensor(e, device='cuda')
        torch.cuda.synchronize(); t0 = time.time()
        w, Z = P.stemr(dt, et, **kw)
        torch.cuda.synchronize(); t1 = time.time()
        st = P.last_stats()
        w = w.cpu().numpy(); Z = Z.cpu().numpy()
        wo, Zo = oracle.stemr(d, e, **kw)
        tn = tnorm1(d, e)
        lam = np.max(np.abs(w - wo)) / (4 * n * EPS * tn) if len(w) == len(wo) else float('nan')
        res, orth = check_accuracy(d, e, w, Z)
        rg = residuals(d, e, w, Z); ro = residuals(d, e, wo, Zo)
        ok = dk_comparable(wo, rg, ro)
        vd = float(np.max(vec_diff_signfree(Z[:, ok], Zo[:, ok]))) if ok.any() else 0.0
        print(f"{name:14s} n={n:6d} m={len(w):6d}/{len(wo):6d} t={1e3*(t1-t0):8.2f}ms lam={lam:.3e} res={res:.3e} orth={orth:.3e} vec={vd:.2e} ({ok.sum()} cmp) "
              f"nodes={st['nodes']} lv={st['levels']} rqc={st['rqc_iters']} fb={st['rqc_fallbacks']} safe={st['safe_resweeps']} ms={st['ms_root']:.2f}/{st['ms_tree']:.2f}/{st['ms_vectors']:.2f}", flush=True)
    except Exception as ex:
        print(f"{name}: EXC {ex}", flush=True)
        traceback.print_exc()
