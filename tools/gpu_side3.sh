#!/bin/bash
# side-stream choice (idle, else oldest launch) + equal pieces; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-s}
mkdir -p gpurun_out
bash tools/gpu_envsweep.sh $T random_20000 - MRRR_SIDE_RR=1 MRRR_NSIDE=5 MRRR_NSIDE=6 - MRRR_SIDE_RR=1 MRRR_NSIDE=5 MRRR_NSIDE=6 MRRR_NSIDE=5,MRRR_PIECE_DIV=5 MRRR_PIECE_DIV=3
bash tools/gpu_envsweep.sh $T glued_wilkinson_21000 - MRRR_NSIDE=5
bash tools/gpu_envsweep.sh $T random_100000 - MRRR_NSIDE=5
bash tools/gpu_envsweep.sh $T clement_50000 - MRRR_NSIDE=5
timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline4.txt
MRRR_NSIDE=5 timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline5.txt
exit 0
