#!/bin/bash
# per-kernel executed FP64 instructions, DRAM bytes and durations (ncu metric capture) of bench.py's
# config $2 (default random_20000); tag $1.  Then: python tools/kernel_table.py gpurun_out/$1_kt.csv profiles/r02/kernel_table_<cfg>.json
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CFG=${2:-random_20000}
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --config $CFG"
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
timeout 600 $CMD > gpurun_out/$1_plain.log 2>&1 && \
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/$1_kt.csv $CMD > gpurun_out/$1_ncu.log 2>&1
exit 0
