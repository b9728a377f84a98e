#!/bin/bash
# round-2 final evidence run
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02f
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=12 > $O/pytest_gpu.log 2>&1
echo "rc=$?" >> $O/pytest_gpu.log; tail -n 4 $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
echo "bench rc=$?"; tail -n 6 $O/bench_cfg5.err; cut -c1-900 $O/bench_cfg5.json
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg5.json 2> $O/bench_ref_cfg5.err
echo "ref rc=$?"
for w in cfg4 cfg3 cfg2; do
  timeout 1200 python bench.py --workload $w --no-kernels > $O/bench_$w.json 2> $O/bench_$w.err
  echo "$w rc=$?"; cut -c1-400 $O/bench_$w.json
done
timeout 280 python bench.py --steps 1 --warmup 1 --profile-cycles 40 --no-e2e --no-cpu --no-kernels > $O/plain_launches.log 2>&1 &&
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 1 --warmup 1 --profile-cycles 40 --no-e2e --no-cpu --no-kernels > $O/ncu_launches.log 2>&1
tail -n 3 $O/ncu_launches.log
