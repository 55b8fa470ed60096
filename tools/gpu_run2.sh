#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
MRRR_TRACE=1 timeout 300 python tools/diag_orth.py random_20000 > gpurun_out/r2_random.log 2>&1
MRRR_TRACE=1 MRRR_DEBUG=1 timeout 300 python tools/diag_orth.py clement_50000_subset > gpurun_out/r2_clem.log 2> gpurun_out/r2_clem.err
MRRR_DEBUG=1 timeout 300 python tools/diag_orth.py glued_wilkinson_21000 > gpurun_out/r2_glued.log 2> gpurun_out/r2_glued.err
gzip -f gpurun_out/r2_clem.err gpurun_out/r2_glued.err
exit 0
