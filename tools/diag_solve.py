"""Run one workload through the GPU solver (test tooling): prints stats and
the accuracy metrics; MRRR_DEBUG / MRRR_TRACE_TASK env vars pass through."""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_1205_2107_b200 as P
from paper_1205_2107_b200 import workloads as W
from helpers import check_accuracy
spec = sys.argv[1]
fam, n = spec.split(":")[0], int(spec.split(":")[1])
kw = {}
if len(sys.argv) > 2:
    il, iu = map(int, sys.argv[2].split(".."))
    kw = {"il": il, "iu": iu}
d, e = {"clement": W.clement, "random": lambda n: W.random_uniform(n, 0),
        "glued": lambda n: W.glued_wilkinson(n // 21), "121": W.one_two_one}[fam](n)
w, Z = P.stemr(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda"), **kw)
torch.cuda.synchronize()
st = P.last_stats()
w = w.cpu().numpy(); Z = Z.cpu().numpy()
res, orth = check_accuracy(d, e, w, Z) if len(d) <= 20000 else (float('nan'), float('nan'))
print(spec, kw, "res %.3g orth %.3g" % (res, orth), {k: st[k] for k in ("nodes", "levels", "rqc_iters", "rqc_fallbacks", "ms_total")})
