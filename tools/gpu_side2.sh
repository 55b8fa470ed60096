#!/bin/bash
# side-stream choice by queued tasks + equal pieces; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-s}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "schedule or small or config2 or scratch or host_entry" > gpurun_out/${T}_pytest.log 2>&1
bash tools/gpu_envsweep.sh $T random_20000 - MRRR_SIDE_RR=1 - MRRR_NSIDE=3 MRRR_NSIDE=5 -
bash tools/gpu_envsweep.sh $T glued_wilkinson_21000 -
bash tools/gpu_envsweep.sh $T random_100000 -
bash tools/gpu_envsweep.sh $T clement_50000 -
timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline4.txt
exit 0
