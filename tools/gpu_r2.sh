#!/bin/bash
# round-2 quick cycle: gpu tests (optional), trace of random 20000, bench, launch list; tag = $1, tests = $2 (1/0)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-q}
if [ "${2:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
fi
MRRR_TRACE=1 timeout 300 python tools/diag_orth.py random_20000 > gpurun_out/${T}_random.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for c in ${CONFIGS:-}; do
  timeout 600 python bench.py --steps 3 --warmup 3 --config $c --no-cpu --no-e2e > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench_cfg.err
done
if [ "${LAUNCH:-1}" = "1" ]; then
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu.log 2>&1
fi
exit 0
