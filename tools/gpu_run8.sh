#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/r8_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_vectors|k_bisect|k_zprobe" -s 6 -c 4 -o gpurun_out/r8_prof $CMD > gpurun_out/r8_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r8_ncu.log
exit 0
