cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
PHASES=1 timeout 300 python tools/run_config.py cfg2a --imax 1 > $O/phases_cfg2a.log 2>&1
PHASES=1 timeout 300 python tools/run_config.py cfg2b --imax 1 > $O/phases_cfg2b.log 2>&1
