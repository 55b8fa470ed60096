cd "$GRAFT_REPO_ROOT" || cd /root/repo
# GPU tests, then every BASELINE config through bench.py (no cpu/e2e legs); tag = $1
mkdir -p gpurun_out
T=${1:-cfg}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
for c in random_20000 glued_wilkinson_21000 one_two_one_2000 clement_50000_subset clement_50000; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench_1e5.json 2> gpurun_out/${T}_bench_1e5.err
exit 0
