cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/early.txt
python tools/trace_run.py random_20000 2 2> gpurun_out/tr2_early12.txt
for eb in 0 12 10 8 14; do
  MRRR_EARLY_BITS=$eb timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('early', $eb, round(d['ms_per_step'],2), d['phases_ms'], d['tree'])" >> gpurun_out/early.txt
done
for cfg in random_100000 clement_50000 glued_wilkinson_21000; do
for eb in 0 12; do
  MRRR_EARLY_BITS=$eb timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$cfg early', $eb, round(d['ms_per_step'],2), d['phases_ms'], d['tree'])" >> gpurun_out/early.txt
done
done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/early_tests.txt 2>&1
tail -3 gpurun_out/early_tests.txt
exit 0
