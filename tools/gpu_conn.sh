#!/bin/bash
# 32 hardware queues (library default since set F): side-stream count per config; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-c}
mkdir -p gpurun_out
bash tools/gpu_envsweep.sh $T random_20000 CUDA_DEVICE_MAX_CONNECTIONS=8 - MRRR_NSIDE=6 MRRR_NSIDE=8 MRRR_NSIDE=8,MRRR_PIECE_DIV=3 MRRR_NSIDE=8,MRRR_PIECE_DIV=6
bash tools/gpu_envsweep.sh $T glued_wilkinson_21000 CUDA_DEVICE_MAX_CONNECTIONS=8 - MRRR_NSIDE=6 MRRR_NSIDE=8
bash tools/gpu_envsweep.sh $T clement_50000 CUDA_DEVICE_MAX_CONNECTIONS=8 - MRRR_NSIDE=6 MRRR_NSIDE=8
bash tools/gpu_envsweep.sh $T clement_50000_subset CUDA_DEVICE_MAX_CONNECTIONS=8 - MRRR_NSIDE=6 MRRR_NSIDE=8
bash tools/gpu_envsweep.sh $T random_100000 CUDA_DEVICE_MAX_CONNECTIONS=8 - MRRR_NSIDE=6 MRRR_NSIDE=8
exit 0
