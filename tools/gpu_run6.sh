#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r6_pytest.log 2>&1
MRRR_TRACE=1 timeout 300 python tools/diag_orth.py random_20000 > gpurun_out/r6_random.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r6_bench.json 2> gpurun_out/r6_bench.err
exit 0
