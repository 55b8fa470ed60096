#!/bin/bash
# Full measurement pass (round-end style): bench lines, launch list, ncu of the top kernels, clocks.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-m}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${T}_nvidia_smi.txt 2>&1
(nproc; lscpu | grep "Model name") > gpurun_out/${T}_host.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --steps 3 --warmup 3 --config random_100000 --no-cpu > gpurun_out/${T}_bench_1e5.json 2> gpurun_out/${T}_bench_1e5.err
for c in one_two_one_2000 glued_wilkinson_21000 clement_50000_subset clement_50000; do
  timeout 600 python bench.py --steps 3 --warmup 3 --config $c --no-cpu --no-e2e > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench_cfg.err
done
timeout 600 python bench.py --steps 3 --warmup 3 --impl reference > gpurun_out/${T}_bench_ref.json 2>> gpurun_out/${T}_bench_cfg.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1 && \
for k in k_wvectors_split:9 k_child_step:7 regex:k_refine_warp:9; do
  name=${k%:*}; skip=${k##*:}; tag=${name#regex:}
  timeout 900 ncu --set full --clock-control none --import-source on -k $name -s $skip -c 1 -o gpurun_out/${T}_prof_$tag $CMD > gpurun_out/${T}_ncu_full_$tag.log 2>&1
done
echo "done rc=$?" >> gpurun_out/${T}_ncu_full.log
exit 0
