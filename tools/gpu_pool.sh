cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -k "scratch_cap or workspace or schedule" > gpurun_out/pool_tests.txt 2>&1
tail -3 gpurun_out/pool_tests.txt
for cfg in "MRRR_CK_GB=4 MRRR_CS_GB=16" "MRRR_CK_GB=16 MRRR_CS_GB=4" "MRRR_CK_GB=2 MRRR_CS_GB=16" "MRRR_CK_GB=16 MRRR_CS_GB=2" "MRRR_CK_GB=3 MRRR_CS_GB=3"; do
env $cfg timeout 900 python bench.py --config random_100000 --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],1), round(d['memory']['pool_bytes']/1e9,2), round(d['memory']['workspace_bytes']/1e9,2), d['phases_ms'])" >> gpurun_out/pool_sweep.txt
done
exit 0
