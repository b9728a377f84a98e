cd $GRAFT_REPO_ROOT
O=gpurun_out
for i in 1 2; do
PHASES=1 timeout 300 python tools/run_config.py cfg2a --imax 1 > $O/ab_new_$i.log 2>&1
GB_LIB_PATH=$PWD/tools/ab/libold.so PHASES=1 timeout 300 python tools/run_config.py cfg2a --imax 1 > $O/ab_old_$i.log 2>&1
done
