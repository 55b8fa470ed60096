#!/bin/bash
# GPU tests, then the headline bench with its e2e leg at n=20000 and n=1e5; tag = $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-e2e}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu > gpurun_out/${T}_bench_1e5.json 2> gpurun_out/${T}_bench_1e5.err
exit 0
