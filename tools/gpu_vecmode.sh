cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-vm}
for cm in 0 1; do
  export MRRR_VEC_MODE=$cm
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_$cm.json 2> gpurun_out/${T}_bench_$cm.err
  for w in glued_wilkinson_21000 clement_50000; do
    timeout 600 python bench.py --config $w --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench_${w}_$cm.json 2> gpurun_out/${T}_bench_${w}_$cm.err
  done
  timeout 900 python bench.py --config random_100000 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench1e5_$cm.json 2> gpurun_out/${T}_bench1e5_$cm.err
done
exit 0
