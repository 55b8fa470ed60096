cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-r58}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
for p in 0 1; do
  MRRR_TREE_PRIO=$p timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_p$p.json 2> gpurun_out/${T}_bench_p$p.err
  MRRR_TREE_PRIO=$p timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench1e5_p$p.json 2> gpurun_out/${T}_bench1e5_p$p.err
done
exit 0
