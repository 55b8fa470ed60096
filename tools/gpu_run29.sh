#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/r29_mem.txt
MRRR_TRACE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "config5" --timeout 900 -p no:cacheprovider > gpurun_out/r29_cfg5.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "not config5" > gpurun_out/r29_pytest.log 2>&1
exit 0
