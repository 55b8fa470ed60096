# usage: bash tools/gpu_sanitize.sh <tool>   (one compute-sanitizer tool per call)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
t=${1:-memcheck}
extra=""
[ "$t" = "memcheck" ] && extra="--leak-check no"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --target-processes all --print-limit 50 \
  python tools/sanitize_run.py > gpurun_out/sanitize_$t.txt 2>&1
echo "exit $?" >> gpurun_out/sanitize_$t.txt
tail -5 gpurun_out/sanitize_$t.txt
