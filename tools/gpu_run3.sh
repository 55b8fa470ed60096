#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for spec in "clement:20000 1..2000" "clement:6000 1..1500" "clement:50000 1..5000"; do
  tag=$(echo $spec | tr ': .' '___')
  MRRR_DEBUG=1 timeout 300 python tools/diag_solve.py $spec > gpurun_out/r3_$tag.log 2> gpurun_out/r3_$tag.err
  ids=$(grep "fb 1" gpurun_out/r3_$tag.err | head -3 | awk '{print $2}')
  for t in $ids; do
    MRRR_TRACE_TASK=$t timeout 300 python tools/diag_solve.py $spec >> gpurun_out/r3_$tag.trace 2>&1
  done
  gzip -f gpurun_out/r3_$tag.err
done
exit 0
