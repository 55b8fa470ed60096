"""paper_1205_2107_b200 -- B200-native (sm_100a) fp64 MRRR symmetric
tridiagonal eigensolver (the hot path of arXiv 1205.2107, PMRRR).

Public API: :func:`stemr` (see ``mrrr.py``; C ABI in ``include/mrrr.h``).
"""
from .mrrr import (NcclComm, default_opts, last_stats, rqc_histogram, shard_columns, stemr, stemr_dist,  # noqa: F401
                   stemr_host, stemr_nccl, trim_workspace, version)
