#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for pd in ${PDS:-4 2}; do
  for c in random_20000 glued_wilkinson_21000 clement_50000; do
    MRRR_PIECE_DIV=$pd timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu --no-e2e > gpurun_out/$1_${c}_$pd.json 2> gpurun_out/$1_${c}_$pd.err
  done
done
exit 0
