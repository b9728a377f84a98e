cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
rm -f $O/pk_lu.log
for i in 1 2; do timeout 300 python tools/prof_kernels.py lu 16384 half single double exact >> $O/pk_lu.log 2>&1; done
timeout 300 python tools/prof_kernels.py lu 8192 half single double exact >> $O/pk_lu.log 2>&1
PHASES=1 timeout 300 python tools/run_config.py cfg2b --imax 1 > $O/phases_cfg2b.log 2>&1
