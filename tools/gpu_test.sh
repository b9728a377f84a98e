cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
PHASES=1 timeout 300 python tools/run_config.py cfg2a --imax 1 > $O/phases_cfg2a.log 2>&1
for i in 1 2; do
timeout 300 python tools/prof_kernels.py op 8192 single double quad > $O/pk_op8192_$i.log 2>&1
timeout 300 python tools/prof_kernels.py op 16384 half single double > $O/pk_op16384_$i.log 2>&1
done
timeout 600 python tools/run_config.py cfg4 > $O/run_cfg4.log 2>&1
