#!/bin/bash
# round-2 status run: micro tcgemm, operator check, full GPU suite, cfg5 end-to-end
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
(cd tools/micro && timeout 120 ./tcgemm 8192 256; timeout 120 ./tcgemm 16384 256; timeout 120 ./tcgemm 16384 512; timeout 120 ./tcgemm 16384 1024) > gpurun_out/tcgemm.log 2>&1
timeout 300 python tools/op_check.py > gpurun_out/op_check.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 5 gpurun_out/pytest_gpu.log
timeout 1500 python tools/run_config.py cfg5 > gpurun_out/cfg5_full.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_full.log
tail -n 8 gpurun_out/cfg5_full.log
