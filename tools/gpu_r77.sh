cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-r77}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
for i in 1 2; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_a$i.json 2> gpurun_out/${T}_bench_a$i.err
  MRRR_VEC_SPLIT=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_b$i.json 2> gpurun_out/${T}_bench_b$i.err
done
timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench_1e5.json 2> gpurun_out/${T}_bench_1e5.err
timeout 600 python bench.py --config glued_wilkinson_21000 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_glued.json 2> gpurun_out/${T}_bench_glued.err
exit 0
