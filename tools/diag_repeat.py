"""Repeated solves of one workload (test tooling): wall time per call, MRRR_TRACE passes through.
usage: python tools/diag_repeat.py <bench config name> [calls]"""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1205_2107_b200 as P
from paper_1205_2107_b200 import workloads as W
d, e, rng = W.make(sys.argv[1])
kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
k = len(d) if rng is None else rng[1] - rng[0] + 1
w = torch.empty(k, dtype=torch.float64, device="cuda")
Z = torch.empty((k, len(d)), dtype=torch.float64, device="cuda")
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    P.stemr(dt, et, w=w, Z=Z, **kw)
    torch.cuda.synchronize()
    st = P.last_stats()
    print(f"call {i}: wall {1e3 * (time.perf_counter() - t):.2f} ms  device total {st['ms_total']:.2f}", flush=True)
