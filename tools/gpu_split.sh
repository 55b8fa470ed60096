#!/bin/bash
# split-count experiment: bench per MRRR_SPLIT, trace, parity tests; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-sp}
for sp in ${SPLITS:-0 1 2}; do
  for c in ${CONFIGS:-random_20000}; do
    MRRR_SPLIT=$sp timeout 600 python bench.py --steps 10 --warmup 3 --config $c --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('split $sp $c', round(d['ms_per_step'],2), d['phases_ms'])" >> gpurun_out/${T}_split.txt
  done
done
MRRR_SPLIT=${TRACE_SPLIT:-1} timeout 300 python tools/trace_run.py random_20000 2 2> gpurun_out/${T}_trace2.txt
if [ "${TESTS:-1}" = "1" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
fi
exit 0
