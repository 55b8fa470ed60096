"""Projected strong scaling of mrrr_stemr_dist from ONE GPU (test tooling):
for P = 1, 2, 4, 8 the P ranks' solves run one after another on this GPU
(the all-gather of w replaced by a local placement, as in
tests/test_gpu_dist.py), each timed with CUDA events after a warm-up; the
projected P-GPU step is the slowest rank's time (no NVLink traffic besides
the w all-gather, which is m * 8 bytes).  Prints one JSON line per P.
usage: python tools/virtual_scaling.py [config] [reps]"""
import json, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
import paper_1205_2107_b200 as P
from paper_1205_2107_b200 import workloads as W
from test_gpu_dist import local_allgather

cfg = sys.argv[1] if len(sys.argv) > 1 else "random_20000"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
d, e, rng = W.make(cfg)
kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
out = {}
for nr in (1, 2, 4, 8):
    times = []
    for r in range(nr):
        cb = local_allgather(r, nr)
        best = None
        for it in range(reps + 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            w_all, Zl, c0 = P.stemr_dist(dt, et, rank=r, nranks=nr, allgather=cb, **kw)
            b.record()
            torch.cuda.synchronize()
            if it > 0:
                ms = a.elapsed_time(b)
                best = ms if best is None else min(best, ms)
            del Zl
        st = P.last_stats()
        times.append(best)
    m = w_all.shape[0]
    out[nr] = max(times)
    print(json.dumps({"config": cfg, "nranks": nr, "rank_ms": [round(t, 2) for t in times],
                      "projected_step_ms": round(max(times), 2),
                      "projected_speedup": round(out[1] / max(times), 2),
                      "projected_pairs_per_s": round(m / (max(times) / 1e3))}), flush=True)
