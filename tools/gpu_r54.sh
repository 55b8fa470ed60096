cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r54_pytest.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r54_bench_$i.json 2> gpurun_out/r54_bench_$i.err; done
MRRR_RW_M=4 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r54_bench_m4.json 2> gpurun_out/r54_bench_m4.err
exit 0
