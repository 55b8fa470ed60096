cd "$GRAFT_REPO_ROOT" || cd /root/repo
for wg in 64 16 4; do MRRR_INT_WG=$wg STRATS=1 timeout 900 python tools/diag_strategy.py random_20000 clement_50000 >> gpurun_out/r2o_strat.jsonl 2>> gpurun_out/r2o_strat.err; done
STRATS=0,1 timeout 900 python tools/diag_strategy.py random_100000 >> gpurun_out/r2o_strat.jsonl 2>> gpurun_out/r2o_strat.err
exit 0
