cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-r67}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
for c in random_20000 one_two_one_2000 glued_wilkinson_21000 clement_50000_subset; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
exit 0
