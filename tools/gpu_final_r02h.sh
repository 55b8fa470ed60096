#!/bin/bash
# round-2 closing set, part 1 (after a default change): gpu tests, per-kernel ncu metrics and launch list of
# the bench command, orthogonality of three configs, timeline; tag $1.  Part 2 is tools/gpu_measure_r02.sh.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-h}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
tail -2 gpurun_out/${T}_pytest.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_kt.csv $CMD > gpurun_out/${T}_ncu_kt.log 2>&1
for c in random_20000 glued_wilkinson_21000 clement_50000; do
  timeout 600 python tools/diag_orth.py $c 2>&1 | grep -v "^\[mrrr" | tail -6 >> gpurun_out/${T}_orth.txt
done
cat gpurun_out/${T}_orth.txt
timeout 300 python tools/timeline_run.py random_20000 2> gpurun_out/${T}_timeline.txt
exit 0
