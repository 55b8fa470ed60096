#!/bin/bash
# side-stream selection / count sweep; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-s}
mkdir -p gpurun_out
bash tools/gpu_envsweep.sh $T random_20000 MRRR_SIDE_RR=1 - MRRR_NSIDE=6 MRRR_NSIDE=8 MRRR_SIDE_RR=1,MRRR_NSIDE=8 - MRRR_NSIDE=3
bash tools/gpu_envsweep.sh $T glued_wilkinson_21000 MRRR_SIDE_RR=1 - MRRR_NSIDE=8
bash tools/gpu_envsweep.sh $T random_100000 MRRR_SIDE_RR=1 - MRRR_NSIDE=8
timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline4.txt
MRRR_NSIDE=8 timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline8.txt
exit 0
