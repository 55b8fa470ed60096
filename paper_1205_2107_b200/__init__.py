"""paper_1205_2107_b200 -- B200-native (sm_100a) fp64 MRRR symmetric
tridiagonal eigensolver (the hot path of arXiv 1205.2107, PMRRR).

Public API: :func:`stemr` (see ``mrrr.py``; C ABI in ``include/mrrr.h``).
"""
from .mrrr import default_opts, last_stats, stemr, stemr_host, trim_workspace, version  # noqa: F401
