#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02l
mkdir -p $O
for w in cfg4 cfg3; do
  timeout 1200 python bench.py --workload $w --no-kernels > $O/bench_$w.json 2> $O/bench_$w.err
  echo "$w rc=$?"; cut -c1-300 $O/bench_$w.json
done
python __graft_entry__.py --smoke > $O/smoke.log 2>&1; tail -n 2 $O/smoke.log
