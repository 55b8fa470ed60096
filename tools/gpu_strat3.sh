cd "$GRAFT_REPO_ROOT" || cd /root/repo
FULL=1 STRATS=1 timeout 900 python tools/diag_strategy.py clement_50000 random_20000 > gpurun_out/r2t_strat.jsonl 2> gpurun_out/r2t_strat.err
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1
exit 0
