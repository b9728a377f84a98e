cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_cfg3.py > gpurun_out/diag_cfg3.log 2>&1
PHASES=1 timeout 300 python tools/run_config.py cfg2a --imax 1 > gpurun_out/phases_cfg2a.log 2>&1
PHASES=1 timeout 300 python tools/run_config.py cfg2b --imax 1 > gpurun_out/phases_cfg2b.log 2>&1
STEPS=1 timeout 300 python tools/prof_step.py 8192 single double quad 100 20 > gpurun_out/prof_8192.log 2>&1
STEPS=1 timeout 300 python tools/prof_step.py 16384 half single double 200 30 > gpurun_out/prof_16384.log 2>&1
