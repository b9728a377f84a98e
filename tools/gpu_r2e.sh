#!/bin/bash
# round-2: blocked tensor LU, tagged MGS reductions, packed hqr2, cfg5
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python tools/lu_tc_check.py 2048 4096 16384 > gpurun_out/lu_tc.log 2>&1
echo "rc=$?" >> gpurun_out/lu_tc.log
cat gpurun_out/lu_tc.log
PHASES=1 timeout 600 python tools/run_config.py cfg5 --n 4096 --max-cycles 2 > gpurun_out/cfg5_4096_ph.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_4096_ph.log
tail -n 22 gpurun_out/cfg5_4096_ph.log
timeout 1500 python -m pytest tests -m gpu -q -rs -x --deselect tests/test_gpu_configs.py::test_config2_cluster_team --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 25 gpurun_out/pytest_gpu.log
PHASES=1 timeout 1500 python tools/run_config.py cfg5 --max-cycles 4 > gpurun_out/cfg5_c4.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_c4.log
tail -n 25 gpurun_out/cfg5_c4.log
