#!/bin/bash
# A/B of a library variant built elsewhere (tmp_variants/$2) against the in-tree build; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=$1; V=$2; CFG=${3:-random_20000}
mkdir -p gpurun_out
cp paper_1205_2107_b200/libmrrr_b200.so /tmp/lib_base.so
for rep in 1 2; do
  cp /tmp/lib_base.so paper_1205_2107_b200/libmrrr_b200.so
  bash tools/gpu_envsweep.sh ${T} $CFG -
  cp tmp_variants/$V paper_1205_2107_b200/libmrrr_b200.so
  bash tools/gpu_envsweep.sh ${T}_v $CFG -
done
cp /tmp/lib_base.so paper_1205_2107_b200/libmrrr_b200.so
exit 0
