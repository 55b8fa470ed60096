"""RQC trajectories of the slowest lanes (MRRR_DEBUG_RQC; diagnostic): solves a random matrix with the
un-split vector kernels (which print every RQC step) and prints the steps of the eigenpairs that took
the most factorizations.  usage: python tools/diag_rqc_tail.py [n] [seed]  (stdout of the kernels is
read back from a pipe)"""
import os
import re
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.getcwd())
    import torch
    import paper_1205_2107_b200 as P
    from paper_1205_2107_b200 import workloads as W
    n, seed = int(sys.argv[2]), int(sys.argv[3])
    d, e = W.random_uniform(n, seed)
    w, Z = P.stemr(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda"))
    torch.cuda.synchronize()
    print("HIST", P.rqc_histogram())
    sys.exit(0)

n = sys.argv[1] if len(sys.argv) > 1 else "3000"
seed = sys.argv[2] if len(sys.argv) > 2 else "4"
env = dict(os.environ, MRRR_DEBUG_RQC="1", MRRR_VEC_SPLIT="0", MRRR_VEC_PSPLIT="0", MRRR_VEC_MODE="1")
out = subprocess.run([sys.executable, __file__, "--child", n, seed], env=env, capture_output=True, text=True).stdout
steps = {}
for ln in out.splitlines():
    m = re.match(r"rqc task (\d+) it (\d+) (.*)", ln)
    if m:
        steps.setdefault(int(m.group(1)), []).append((int(m.group(2)), m.group(3)))
    elif ln.startswith("HIST"):
        print(ln)
worst = sorted(steps.items(), key=lambda kv: -len(kv[1]))[:6]
for t, st in worst:
    print(f"--- task {t}: {len(st)} steps")
    for it, rest in st:
        print(f"  it {it} {rest}")
