#!/bin/bash
# round-2 final evidence run (after the GEMV column passes / cluster-kernel diet)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02k
mkdir -p $O
timeout 600 python tools/op_check.py > $O/op_check.log 2>&1; cat $O/op_check.log
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=8 > $O/pytest_gpu.log 2>&1
echo "rc=$?" >> $O/pytest_gpu.log; tail -n 4 $O/pytest_gpu.log
timeout 900 python bench.py --workload cfg2 --no-kernels > $O/bench_cfg2.json 2> $O/bench_cfg2.err; cut -c1-260 $O/bench_cfg2.json
timeout 1500 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
echo "bench rc=$?"; tail -n 5 $O/bench_cfg5.err; cut -c1-400 $O/bench_cfg5.json
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg5.json 2> $O/bench_ref_cfg5.err
echo "ref rc=$?"
PHASES=1 timeout 900 python tools/run_config.py cfg5 --max-cycles 3 > $O/cfg5_c3.log 2>&1
grep -E "^ +(1[0-9]|2[0-9]|4[0-9]|6[0-9])->" $O/cfg5_c3.log | head -8
