#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02i
mkdir -p $O
PHASES=1 timeout 600 python tools/run_config.py cfg5 --n 4096 --max-cycles 3 > $O/cfg5_4096_ph.log 2>&1
echo "rc=$?" >> $O/cfg5_4096_ph.log; grep -E "^ +(4[0-9]|6[0-9])->" $O/cfg5_4096_ph.log | head -5; tail -n 4 $O/cfg5_4096_ph.log
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_kernels.py -m gpu -q -x -k "config5 or grid_team or inner_solver" > $O/pytest_sub.log 2>&1
tail -n 5 $O/pytest_sub.log
