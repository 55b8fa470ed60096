"""RQC trajectory of a zero-diagonal tridiagonal (MRRR_DEBUG_RQC; diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1205_2107_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
os.environ["MRRR_RW_ROOT_M"] = sys.argv[2] if len(sys.argv) > 2 else "2"
os.environ["MRRR_DEBUG_RQC"] = "1"
d = np.zeros(n); e = np.ones(n - 1)
w, Z = P.stemr(torch.tensor(d, device="cuda"), torch.tensor(e, device="cuda"))
torch.cuda.synchronize()
print(w.cpu().numpy())
