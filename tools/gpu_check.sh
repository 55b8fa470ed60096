cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/check_tests.txt 2>&1
tail -3 gpurun_out/check_tests.txt
rm -f gpurun_out/check.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('20k', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],1), d['phases_ms'], d['roofline']['frac'])" >> gpurun_out/check.txt
for c in random_100000:2 glued_wilkinson_21000:3; do
cfg=${c%%:*}; st=${c##*:}
timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],2), d['phases_ms'])" >> gpurun_out/check.txt
done
exit 0
