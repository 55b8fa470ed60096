#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out/dump_clem20k
MRRR_DUMP=gpurun_out/dump_clem20k timeout 300 python tools/diag_solve.py clement:20000 1..2000 > gpurun_out/r4.log 2>&1
exit 0
