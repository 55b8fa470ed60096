#!/bin/bash
# bench.py under several environment settings: $1 tag, $2 config, then "VAR=val[,VAR=val]" settings ("-" = default)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=$1; CFG=$2; shift 2
for setting in "$@"; do
  envs=""
  [ "$setting" != "-" ] && envs=$(echo "$setting" | tr ',' ' ')
  ms=$(env $envs timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --config $CFG 2>>gpurun_out/${T}_sweep.err | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(round(d['ms_per_step'],2), d['phases_ms'], d['tree']['levels'])")
  echo "$CFG [$setting] $ms" >> gpurun_out/${T}_sweep.txt
done
exit 0
