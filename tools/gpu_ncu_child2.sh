cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/r2x_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_child_step2 -s 5 -c 1 -o gpurun_out/r2x_child2 $CMD > gpurun_out/r2x_ncu1.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/r2x_plain.log').read().splitlines()[-1]);print(d['ms_per_step'])" >> gpurun_out/r2x_ncu1.log
exit 0
