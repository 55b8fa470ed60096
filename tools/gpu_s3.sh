#!/bin/bash
# session-3 check: gpu tests, default bench, level trace of random 20000; tag = $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-s3}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 300 python tools/trace_run.py random_20000 2 2> gpurun_out/${T}_trace2.txt
exit 0
