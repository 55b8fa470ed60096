"""Device timeline of one solve (MRRR_TIMELINE=1, stderr) after warm-up
(profiling tooling).  usage: python tools/timeline_run.py config"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1205_2107_b200 as P  # noqa: E402
from paper_1205_2107_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "random_20000"
d, e, rng = W.make(cfg)
kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
dt = torch.tensor(d, device="cuda")
et = torch.tensor(e, device="cuda")
for _ in range(3):
    w, Z = P.stemr(dt, et, **kw)
    del w, Z
torch.cuda.synchronize()
os.environ["MRRR_TIMELINE"] = "1"
w, Z = P.stemr(dt, et, **kw)
torch.cuda.synchronize()
