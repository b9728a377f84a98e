cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/bench_cfg2.log
timeout 600 python bench.py --workload cfg3 --no-cpu > gpurun_out/bench_cfg3.log 2>&1; echo "rc $?" >> gpurun_out/bench_cfg3.log
