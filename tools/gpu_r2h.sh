#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python tools/crash_hunt.py > gpurun_out/crash_hunt.log 2>&1
cat gpurun_out/crash_hunt.log
(cd tools/micro && for a in "16384 1024 1" "16384 1024 2" "16384 2048 1" "8192 1024 1"; do timeout -k 10 90 ./tcgemm $a; echo "rc=$?"; done) > gpurun_out/tcgemm4.log 2>&1
cat gpurun_out/tcgemm4.log
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "inner_solver or tensor" > gpurun_out/pytest_sub.log 2>&1
tail -n 15 gpurun_out/pytest_sub.log
