#!/bin/bash
# round-end dress rehearsal in the driver's order: smoke(), the default bench line, the reference arm; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-dress}
mkdir -p gpurun_out
( timeout 600 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/${T}_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/${T}_smoke.txt
for i in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/${T}_bench_$i.json 2> gpurun_out/${T}_bench_$i.err
  echo "bench $i rc=$?" >> gpurun_out/${T}_smoke.txt
done
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
echo "ref rc=$?" >> gpurun_out/${T}_smoke.txt
cat gpurun_out/${T}_smoke.txt
exit 0
