cd $GRAFT_REPO_ROOT
O=gpurun_out/final3
mkdir -p $O/prof
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_cfg2.log 2>&1; echo "rc $?" >> $O/bench_cfg2.log
timeout 600 python bench.py --workload cfg3 --no-kernels > $O/bench_cfg3.log 2>&1; echo "rc $?" >> $O/bench_cfg3.log
timeout 900 $NCU --set full --clock-control none -k regex:k_lu_team -c 1 -o $O/prof/ncu_lu_tensor -f \
  python tools/prof_kernels.py lu 16384 half single double tensor > $O/prof/ncu_lu_tensor.log 2>&1
$NCU -i $O/prof/ncu_lu_tensor.ncu-rep --page details --csv > $O/prof/ncu_lu_tensor_details.csv 2>&1
$NCU -i $O/prof/ncu_lu_tensor.ncu-rep --page raw --csv > $O/prof/ncu_lu_tensor_raw.csv 2>&1
rm -f $O/prof/ncu_lu_tensor.ncu-rep
