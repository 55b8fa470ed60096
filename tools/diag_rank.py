"""One virtual rank of a sharded solve (test tooling; MRRR_TRACE passes through).
usage: python tools/diag_rank.py <config> <rank> <nranks>"""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
import paper_1205_2107_b200 as P
from paper_1205_2107_b200 import workloads as W
from test_gpu_dist import local_allgather
d, e, rng = W.make(sys.argv[1])
r, nr = int(sys.argv[2]), int(sys.argv[3])
dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
for it in range(2):
    w_all, Zl, c0 = P.stemr_dist(dt, et, rank=r, nranks=nr, allgather=local_allgather(r, nr))
    torch.cuda.synchronize()
    print("call", it, P.last_stats()["ms_total"], flush=True)
    del Zl
