python tools/trace_run.py random_20000 1 2> gpurun_out/tr1.txt
python tools/trace_run.py random_20000 2 2> gpurun_out/tr2.txt
MRRR_VEC_MODE=1 python tools/trace_run.py random_20000 1 2> gpurun_out/tr1v.txt
MRRR_VEC_MODE=1 python tools/trace_run.py random_20000 2 2> gpurun_out/tr2v.txt
