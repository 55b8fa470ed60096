#!/bin/bash
# quick GPU cycle: tests, random-20000 trace, bench; tag = $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-q}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
MRRR_TRACE=1 timeout 300 python tools/diag_orth.py random_20000 > gpurun_out/${T}_random.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu.log 2>&1
exit 0
