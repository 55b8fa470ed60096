"""Small solves for compute-sanitizer (test tooling): every kernel of the
path on inputs that reach the tree (several levels), the split matrix path,
INDEX / VALUE ranges, the RQC fallback (1-2-1), the host entry, values only.
usage: compute-sanitizer --tool <memcheck|racecheck|synccheck|initcheck> python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_2107_b200 as P  # noqa: E402
from paper_1205_2107_b200 import workloads as W  # noqa: E402


def run(d, e, **kw):
    dt = torch.tensor(np.asarray(d, float), device="cuda")
    et = torch.tensor(np.asarray(e, float) if len(e) else np.zeros(1), device="cuda")
    w, Z = P.stemr(dt, et, **kw)
    torch.cuda.synchronize()
    return w, Z


cases = []
d, e = W.glued_wilkinson(40)
cases.append(("glued_40", d, e, {}))
d, e = W.random_uniform(1200, 3)
cases.append(("random_1200", d, e, {}))
cases.append(("random_1200_idx", d, e, {"il": 100, "iu": 400}))
d, e = W.clement(800)
cases.append(("clement_800", d, e, {}))
d, e = W.one_two_one(600)
cases.append(("one_two_one_600", d, e, {}))
d = np.concatenate([W.random_uniform(300, 4)[0], W.random_uniform(200, 5)[0]])
e = np.concatenate([W.random_uniform(300, 4)[1], [0.0], W.random_uniform(200, 5)[1]])
cases.append(("split_500", d, e, {}))
for name, d, e, kw in cases:
    w, Z = run(d, e, **kw)
    print(name, "m", w.shape[0], "levels", P.last_stats()["levels"], flush=True)
d, e = W.random_uniform(1200, 3)
w, _ = run(d, e, vectors=False)
print("values only ok", flush=True)
w2, Z2 = P.stemr_host(torch.tensor(d).pin_memory(), torch.tensor(e).pin_memory(),
                      Z=torch.empty((1200, 1200), dtype=torch.float64).pin_memory())
# the multi-GPU protocol on virtual ranks (host-thread all-gathers), 2 ranks
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from vranks import VirtualRanks  # noqa: E402
out = VirtualRanks(2).run(d, e)
assert all(o[0] == 0 for o in out), [o[0] for o in out]
print("dist 2 ok", flush=True)
print("host entry ok", flush=True)
