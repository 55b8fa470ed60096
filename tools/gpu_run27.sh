#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
MRRR_DEBUG_TASKS=1 timeout 600 python tools/diag_orth.py glued_wilkinson_21000 > gpurun_out/r27_glued.log 2> gpurun_out/r27_glued.err
gzip -f gpurun_out/r27_glued.err
exit 0
