#!/bin/bash
# round-2 session-4 check: gpu tests and the bench lines at HEAD; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-e}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
bash tools/gpu_measure_r02.sh ${T}
timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline.txt
MRRR_TRACE=2 timeout 300 python tools/trace_run.py random_100000 2 2> gpurun_out/${T}_trace2_1e5.txt
exit 0
