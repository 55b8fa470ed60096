#!/bin/bash
# the headline bench three times (device leg only): noise check; tag = $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/$1_b$i.json 2> gpurun_out/$1_b$i.err; done
exit 0
