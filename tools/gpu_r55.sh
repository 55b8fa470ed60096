cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-r55}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_$i.json 2> gpurun_out/${T}_bench_$i.err; done
timeout 900 python bench.py --config random_100000 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench1e5.json 2> gpurun_out/${T}_bench1e5.err
MRRR_TRACE=1 timeout 900 python tools/diag_solve.py random:100000 > gpurun_out/${T}_1e5.log 2>&1
exit 0
