#!/bin/bash
# end-to-end (host entry) step under piece schedules that finish columns earlier; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-e}
OUT=gpurun_out/${T}_e2e_sched.txt
rm -f $OUT
for setting in - MRRR_VEC_PAIR=2 MRRR_PIECE_DIV=8 MRRR_PIECE_DIV=16 MRRR_PIECE_DIV=8,MRRR_TREE_SIDE=4 MRRR_PIECE_DIV=16,MRRR_TREE_SIDE=4 MRRR_PIECE_DIV=16,MRRR_TREE_SIDE=4,MRRR_VEC_PAIR=2 MRRR_PIECE_DIV=12,MRRR_NSIDE=6 MRRR_ZB=32,MRRR_PIECE_DIV=16,MRRR_TREE_SIDE=4 -; do
  envs=""
  [ "$setting" != "-" ] && envs=$(echo "$setting" | tr ',' ' ')
  env $envs timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('[$setting]', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), d['e2e']['z_copies_per_step'])" >> $OUT
done
cat $OUT
exit 0
