#!/bin/bash
# round-2 measurement set, part A: the driver's bench lines and the BASELINE configs; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-m}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${T}_nvidia_smi.txt 2>&1
(nproc; lscpu | grep "Model name") > gpurun_out/${T}_host.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
for c in one_two_one_2000 glued_wilkinson_21000 clement_50000_subset clement_50000; do
  timeout 600 python bench.py --steps 3 --warmup 3 --config $c --no-cpu --no-e2e > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench_cfg.err
done
timeout 900 python bench.py --steps 3 --warmup 3 --config random_100000 --no-cpu > gpurun_out/${T}_bench_random_100000.json 2>> gpurun_out/${T}_bench_cfg.err
exit 0
