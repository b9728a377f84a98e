cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O/final
timeout 1200 python bench.py > $O/final/bench_cfg2.log 2>&1; echo "rc $?" >> $O/final/bench_cfg2.log
timeout 600 python bench.py --workload cfg3 --no-kernels > $O/final/bench_cfg3.log 2>&1; echo "rc $?" >> $O/final/bench_cfg3.log
timeout 600 python bench.py --impl reference > $O/final/bench_ref.log 2>&1; echo "rc $?" >> $O/final/bench_ref.log
bash tools/gpu_prof.sh
