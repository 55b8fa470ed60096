cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-r69}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
for hp in 1 0; do
  for c in random_20000 glued_wilkinson_21000; do
    MRRR_HP_STREAM=$hp timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_${c}_$hp.json 2> gpurun_out/${T}_bench_${c}_$hp.err
  done
  MRRR_HP_STREAM=$hp timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench_1e5_$hp.json 2> gpurun_out/${T}_bench_1e5_$hp.err
done
exit 0
