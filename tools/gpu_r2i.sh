#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python tools/crash_hunt.py > gpurun_out/crash_hunt.log 2>&1
cat gpurun_out/crash_hunt.log
PHASES=1 timeout 600 python tools/run_config.py cfg5 --n 4096 --max-cycles 2 > gpurun_out/cfg5_4096_ph.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_4096_ph.log
tail -n 22 gpurun_out/cfg5_4096_ph.log
timeout 900 python tools/lu_tc_check.py 4096 16384 > gpurun_out/lu_tc.log 2>&1
cat gpurun_out/lu_tc.log
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_solve.py tests/test_gpu_kernels.py -m gpu -q -x -k "inner_solver or tensor or config5 or config1 or wellposed or table5 or config2" > gpurun_out/pytest_sub.log 2>&1
tail -n 15 gpurun_out/pytest_sub.log
