#!/bin/bash
# reading 30's interior shift under several weighted-growth bounds (MRRR_INT_WG); tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-iw}
mkdir -p gpurun_out
STRATS=0 timeout 900 python tools/diag_strategy.py random_20000 clement_50000 glued_wilkinson_21000 random_100000 >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
for wg in ${WGS:-2 4 8 64}; do
  STRATS=1 MRRR_INT_WG=$wg timeout 900 python tools/diag_strategy.py random_20000 clement_50000 glued_wilkinson_21000 random_100000 >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
done
exit 0
