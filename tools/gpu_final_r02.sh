#!/bin/bash
# round-2 final set: gpu tests, bench lines (headline + reference arm + configs), then the profile set; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
bash tools/gpu_measure_r02.sh ${T}
VS=${VS:-1} bash tools/gpu_profile_r02b.sh ${T}
timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline.txt
MRRR_TRACE=2 timeout 300 python tools/trace_run.py random_20000 2 2> gpurun_out/${T}_trace2.txt
exit 0
