#!/bin/bash
# vector-kernel shared-memory footprint: library variants tmp_variants/libv_r<ring>_s<maxseg>.so against the built one
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-v}
OUT=gpurun_out/${T}_vsmem.txt
rm -f $OUT
cp paper_1205_2107_b200/libmrrr_b200.so /tmp/base.so
CFGS=${CFGS:-random_20000}
for c in $CFGS; do
for v in base $(ls tmp_variants | sed 's/^lib//; s/\.so$//') base; do
  if [ $v = base ]; then cp /tmp/base.so paper_1205_2107_b200/libmrrr_b200.so; else cp tmp_variants/lib$v.so paper_1205_2107_b200/libmrrr_b200.so; fi
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 4 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],2), d['phases_ms'], d['tree']['vec_items'])" >> $OUT
done
done
cp /tmp/base.so paper_1205_2107_b200/libmrrr_b200.so
cat $OUT
exit 0
