"""Host trace (MRRR_TRACE) of one solve with a given child-shift strategy
(diagnostic).  usage: python tools/trace_strategy.py config strategy level"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1205_2107_b200 as P  # noqa: E402
from paper_1205_2107_b200 import workloads as W  # noqa: E402

cfg, strat, lvl = sys.argv[1], int(sys.argv[2]), sys.argv[3]
d, e, rng = W.make(cfg)
kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
dt, et = torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda")
o = P.default_opts(shift_strategy=strat)
for _ in range(3):
    w, Z = P.stemr(dt, et, opts=o, **kw)
    del w, Z
torch.cuda.synchronize()
os.environ["MRRR_TRACE" if lvl != "tl" else "MRRR_TIMELINE"] = lvl if lvl != "tl" else "1"
w, Z = P.stemr(dt, et, opts=o, **kw)
torch.cuda.synchronize()
print(P.last_stats(), file=sys.stderr)
