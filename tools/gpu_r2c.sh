#!/bin/bash
# round-2 diagnostic: cfg5 crash + new config tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -rs -s -k "config2 or config5 or lu_" > gpurun_out/pytest_cfg.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_cfg.log
tail -n 8 gpurun_out/pytest_cfg.log
timeout 600 python tools/run_config.py cfg5 --n 4096 --max-cycles 3 > gpurun_out/cfg5_4096.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_4096.log
tail -n 6 gpurun_out/cfg5_4096.log
timeout 1200 python tools/run_config.py cfg5 --max-cycles 3 > gpurun_out/cfg5_c3.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_c3.log
tail -n 6 gpurun_out/cfg5_c3.log
if grep -q "rc=1" gpurun_out/cfg5_4096.log; then
  timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/run_config.py cfg5 --n 4096 --max-cycles 2 > gpurun_out/cfg5_san.log 2>&1
  tail -n 40 gpurun_out/cfg5_san.log
fi
