#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for spec in "clement:20000 1..2000" "clement:50000 1..5000" "random:20000" "glued:21000" "clement:50000"; do
  tag=$(echo $spec | tr ': .' '___')
  timeout 300 python tools/diag_solve.py $spec > gpurun_out/r5_$tag.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r5_pytest.log 2>&1
exit 0
