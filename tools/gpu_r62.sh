cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-r62}
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_a.json 2> gpurun_out/${T}_bench_a.err
timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench_random_100000.json 2> gpurun_out/${T}_bench_random_100000.err
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_b.json 2> gpurun_out/${T}_bench_b.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/${T}_smi.txt
exit 0
