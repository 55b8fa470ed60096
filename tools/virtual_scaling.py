"""Projected strong scaling of mrrr_stemr_dist from ONE GPU (test tooling).

For P = 1, 2, 4, 8 the P ranks run as host threads (tests/vranks.py) with
their GPU work serialised between collectives: each rank runs each of its
phases (the work between two all-gathers) alone on the GPU, synchronised at
both ends, and the phase's wall time is recorded.  The projected P-GPU step
is  sum over phases of  max over ranks  of the phase time,  plus a latency
of LAT_US per collective (NVLink/NVSwitch all-gathers of <= 2 n doubles per
rank; B200_PROFILING.md measures 770 GB/s per direction, so the bytes add
< 20 us at n = 1e5).  Synchronising every phase also forces the side-stream
vector pieces of a level to finish inside it, so the projection is
pessimistic against a real multi-GPU run (no overlap across levels), and
P = 1 is measured the same way for the ratio.  The vectors run in one batch
after the tree (MRRR_VEC_MODE=1) for every P, so that a level's phase holds
the level's tree work only.  Ranks are persistent threads (warm workspace).
Prints one JSON line per P.
usage: python tools/virtual_scaling.py [config] [reps] [P list]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ.setdefault("MRRR_VEC_MODE", "1")
import torch  # noqa: E402

from paper_1205_2107_b200 import workloads as W  # noqa: E402
from vranks import VirtualRanks  # noqa: E402

LAT_US = 25.0

cfg = sys.argv[1] if len(sys.argv) > 1 else "random_20000"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
plist = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8]
d, e, rng = W.make(cfg)
kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
base = None
for nr in plist:
    best = None
    for it in range(reps + 1):
        vr = VirtualRanks(nr, timed=True)
        out = vr.run(d, e, **kw)
        assert all(o[0] == 0 for o in out), [o[0] for o in out]
        nph = len(vr.phase_ms[0])
        assert all(len(p) == nph for p in vr.phase_ms), [len(p) for p in vr.phase_ms]
        per_phase = [max(vr.phase_ms[r][k] for r in range(nr)) for k in range(nph)]
        proj = sum(per_phase) + (nph - 1) * LAT_US / 1e3
        rank_tot = [sum(p) for p in vr.phase_ms]
        m = out[0][1].shape[0]
        del out
        torch.cuda.empty_cache()
        if it > 0 and (best is None or proj < best[0]):
            best = (proj, per_phase, rank_tot, m)
    proj, per_phase, rank_tot, m = best
    if base is None:
        base = proj
    print(json.dumps({"config": cfg, "nranks": nr, "phases": len(per_phase),
                      "rank_busy_ms": [round(t, 2) for t in rank_tot],
                      "phase_max_ms": [round(t, 2) for t in per_phase],
                      "projected_step_ms": round(proj, 2),
                      "projected_speedup": round(base / proj, 2),
                      "projected_pairs_per_s": round(m / (proj / 1e3))}), flush=True)
