#!/bin/bash
# round-2 (session 3) measurement set, part B: launch list, per-kernel ncu metrics, ncu --set full of the
# top kernels, projected scaling; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-p}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_kt.csv $CMD > gpurun_out/${T}_ncu_kt.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wvectors_psplit -s 8 -c 1 -o gpurun_out/${T}_prof_wvectors $CMD > gpurun_out/${T}_ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_refine_warp -s 9 -c 1 -o gpurun_out/${T}_prof_refine $CMD > gpurun_out/${T}_ncu_full2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_child_chains3|k_child_step2" -s 4 -c 2 -o gpurun_out/${T}_prof_child $CMD > gpurun_out/${T}_ncu_full3.log 2>&1
if [ "${VS:-1}" = "1" ]; then
timeout 900 python tools/virtual_scaling.py random_20000 2 > gpurun_out/${T}_vs20k.jsonl 2> gpurun_out/${T}_vs20k.err
MRRR_SCRATCH_GB=4 timeout 1500 python tools/virtual_scaling.py random_100000 1 1,2,4,8 > gpurun_out/${T}_vs1e5.jsonl 2> gpurun_out/${T}_vs1e5.err
fi
exit 0
