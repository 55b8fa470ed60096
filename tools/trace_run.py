"""Host trace of one solve (test tooling): warm up, then one call with
MRRR_TRACE=<level> (stderr).  usage: python tools/trace_run.py config level"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1205_2107_b200 as P  # noqa: E402
from paper_1205_2107_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "random_20000"
lvl = sys.argv[2] if len(sys.argv) > 2 else "1"
d, e, rng = W.make(cfg)
kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
dt = torch.tensor(d, device="cuda")
et = torch.tensor(e, device="cuda")
for _ in range(3):
    w, Z = P.stemr(dt, et, **kw)
    del w, Z
torch.cuda.synchronize()
os.environ["MRRR_TRACE"] = lvl
w, Z = P.stemr(dt, et, **kw)
torch.cuda.synchronize()
print(P.last_stats(), file=sys.stderr)
