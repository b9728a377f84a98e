# ncu evidence for this round (one GPU, one process at a time)
cd $GRAFT_REPO_ROOT
O=gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/prof_kernels.py step 1024 single double quad 50 10 4 > $O/pk_step1024.log 2>&1
timeout 300 python tools/prof_kernels.py lu 16384 half single double exact > $O/pk_lu_exact.log 2>&1
timeout 300 python tools/prof_kernels.py lu 16384 half single double tensor > $O/pk_lu_tensor.log 2>&1
timeout 300 python tools/prof_kernels.py step 8192 single double quad 20 4 1 > $O/pk_step8192.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_step -c 1 -o $O/ncu_step1024 -f \
  python tools/prof_kernels.py step 1024 single double quad 50 10 4 > $O/ncu_step1024.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_step -c 1 -o $O/ncu_step8192 -f \
  python tools/prof_kernels.py step 8192 single double quad 20 4 1 > $O/ncu_step8192.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_lu_team -c 1 -o $O/ncu_lu_tensor -f \
  python tools/prof_kernels.py lu 16384 half single double tensor > $O/ncu_lu_tensor.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_launches.log 2>&1
timeout 600 python bench.py --workload cfg3 --no-cpu > $O/bench_cfg3.log 2>&1
