cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/variants2.txt
cp paper_1205_2107_b200/libmrrr_b200.so /tmp/base.so
for v in base 4 8 6 base 8 6 4; do
  if [ $v = base ]; then cp /tmp/base.so paper_1205_2107_b200/libmrrr_b200.so; else cp tmp_variants/libv$v.so paper_1205_2107_b200/libmrrr_b200.so; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d['phases_ms'])" >> gpurun_out/variants2.txt
done
for v in base 8 6; do
  if [ $v = base ]; then cp /tmp/base.so paper_1205_2107_b200/libmrrr_b200.so; else cp tmp_variants/libv$v.so paper_1205_2107_b200/libmrrr_b200.so; fi
  timeout 600 python bench.py --config random_100000 --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('1e5 $v', round(d['ms_per_step'],2), d['phases_ms'])" >> gpurun_out/variants2.txt
done
cp /tmp/base.so paper_1205_2107_b200/libmrrr_b200.so
exit 0
