cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/overlap3.txt
for v in 300 1200 5000; do
  MRRR_PAIR_MAXCL=$v timeout 600 python bench.py --config random_100000 --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('1e5 maxcl', $v, round(d['ms_per_step'],2), d['phases_ms'])" >> gpurun_out/overlap3.txt
done
MRRR_TRACE=1 timeout 600 python tools/trace_run.py random_100000 1 2> gpurun_out/tr1_1e5.txt
exit 0
