cd "$GRAFT_REPO_ROOT" || cd /root/repo
for wg in 64 8 2; do FULL=1 MRRR_INT_WG=$wg STRATS=1 timeout 900 python tools/diag_strategy.py clement_50000 random_20000 >> gpurun_out/r2s_strat.jsonl 2>> gpurun_out/r2s_strat.err; done
exit 0
