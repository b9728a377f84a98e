#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
(cd tools/micro && timeout 120 ./tcgemm 8192 256; timeout 120 ./tcgemm 16384 256; timeout 120 ./tcgemm 16384 512) > gpurun_out/tcgemm.log 2>&1
timeout 300 python tools/cfg2a_h.py > gpurun_out/cfg2a_h.log 2>&1
timeout 300 python tools/op_check.py > gpurun_out/op_check.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 5 gpurun_out/pytest_gpu.log
