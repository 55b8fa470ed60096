cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2e2e2.txt
python -m pytest tests -q -m gpu -k "host" -x 2>&1 | tail -3 >> gpurun_out/r2e2e2.txt
for zg in 4 0 16 64; do
  MRRR_ZGAP=$zg timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('zgap', $zg, round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d['e2e']['z_copies_per_step'])" >> gpurun_out/r2e2e2.txt
done
exit 0
