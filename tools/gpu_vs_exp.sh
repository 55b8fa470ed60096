#!/bin/bash
# virtual-rank scaling at n=1e5 under refinement settings; tag = $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for cm in 0:4 16:4 8:1; do
  MRRR_RW_CHUNK=${cm%%:*} MRRR_RW_M=${cm##*:} timeout 1500 python tools/virtual_scaling.py random_100000 1 > gpurun_out/$1_${cm/:/_}.jsonl 2> gpurun_out/$1_${cm/:/_}.err
done
exit 0
