#!/bin/bash
# refinement chunk-size experiment: bench random 20000 / 1e5 per MRRR_RW_CHUNK; tag = $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-c}
for c in 0 8 16 32; do
  MRRR_RW_CHUNK=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err
done
for c in 0 8 32; do
  MRRR_RW_CHUNK=$c timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench1e5_c$c.json 2> gpurun_out/${T}_bench1e5_c$c.err
done
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
exit 0
