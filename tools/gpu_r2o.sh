#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02g
mkdir -p $O
timeout 600 python tools/op_check.py > $O/op_check.log 2>&1; cat $O/op_check.log
PHASES=1 timeout 900 python tools/run_config.py cfg5 --max-cycles 3 > $O/cfg5_c3.log 2>&1
echo "rc=$?" >> $O/cfg5_c3.log; tail -n 14 $O/cfg5_c3.log
timeout 900 python bench.py --workload cfg2 --no-kernels --no-cpu > $O/bench_cfg2.json 2> $O/bench_cfg2.err; cut -c1-300 $O/bench_cfg2.json
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
echo "rc=$?" >> $O/pytest_gpu.log; tail -n 4 $O/pytest_gpu.log
