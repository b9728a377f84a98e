# round-1 closing run: GPU parity suite, smoke, default bench (cfg2), cfg3 bench,
# launch list of the default bench (ncu, after the bench itself exited 0)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R1END_DIR:-r1end}
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg2.log 2>&1; echo "rc $?" >> $O/bench_cfg2.log
timeout 600 python bench.py --workload cfg3 --no-kernels > $O/bench_cfg3.log 2>&1; echo "rc $?" >> $O/bench_cfg3.log
timeout 1200 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kernels > $O/ncu_launches.log 2>&1
