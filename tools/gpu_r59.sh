cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-r59}
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for w in glued_wilkinson_21000 clement_50000 random_100000; do
  timeout 900 python bench.py --config $w --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
exit 0
