#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r7_pytest.log 2>&1
MRRR_TRACE=1 timeout 300 python tools/diag_orth.py random_20000 > gpurun_out/r7_random.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/r7_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r7_launches.csv $CMD > gpurun_out/r7_ncu.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err
exit 0
