#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out profiles/r02
timeout 900 python tools/crash_hunt.py > gpurun_out/crash_hunt.log 2>&1
cut -c1-600 gpurun_out/crash_hunt.log
tools/micro/fp64peak > profiles/r02/fp64_peak.json 2> gpurun_out/fp64peak.err; cat profiles/r02/fp64_peak.json; cp profiles/r02/fp64_peak.json gpurun_out/
timeout 600 python tools/op_check.py > gpurun_out/op_check.log 2>&1; cat gpurun_out/op_check.log
GB_SWEEP_LA=1 timeout 600 python tools/op_check.py > gpurun_out/op_check_la.log 2>&1; cat gpurun_out/op_check_la.log
PHASES=1 timeout 1500 python tools/run_config.py cfg5 --max-cycles 3 > gpurun_out/cfg5_c3.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_c3.log
tail -n 25 gpurun_out/cfg5_c3.log
