cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r82_bench.json 2> gpurun_out/r82_bench.err
exit 0
