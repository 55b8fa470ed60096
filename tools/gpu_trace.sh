python tools/trace_run.py random_20000 2 2> gpurun_out/tr2.txt
MRRR_CHILD_V1=1 python tools/trace_run.py random_20000 2 2> gpurun_out/tr2_v1.txt
MRRR_CHILD_V1=0 python tools/trace_run.py random_20000 2 2> gpurun_out/tr2_v2.txt
