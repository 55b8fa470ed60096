#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/r34_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_wprobe" -s 7 -c 1 -o gpurun_out/r34_prof $CMD > gpurun_out/r34_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r34_ncu.log
exit 0
