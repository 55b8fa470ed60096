python tools/trace_run.py random_20000 2 2> gpurun_out/tr2.txt
MRRR_RW_END=2 python tools/trace_run.py random_20000 2 2> gpurun_out/tr2_end.txt
MRRR_RW_CHUNK=4 python tools/trace_run.py random_20000 2 2> gpurun_out/tr2_c4.txt
MRRR_RW_M=2 python tools/trace_run.py random_20000 2 2> gpurun_out/tr2_m2.txt
