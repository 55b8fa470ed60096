cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/r2j_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_child_step -s 5 -c 1 -o gpurun_out/r2j_child0 $CMD > gpurun_out/r2j_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_root_chain_warp -s 1 -c 1 -o gpurun_out/r2j_rootchain $CMD > gpurun_out/r2j_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_refine_warp<1>" -s 9 -c 1 -o gpurun_out/r2j_refine4 $CMD > gpurun_out/r2j_ncu3.log 2>&1
exit 0
