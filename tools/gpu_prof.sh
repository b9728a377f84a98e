# ncu evidence for this round (one GPU, one process at a time); reports are
# summarised on the box (details/raw csv) and the .ncu-rep files removed so
# gpurun_out stays small
cd $GRAFT_REPO_ROOT
O=gpurun_out/prof
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
summ() {  # $1 = report basename
  $NCU -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>&1
  $NCU -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>&1
  $NCU -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_source.csv 2>&1
  gzip -f $O/$1_source.csv
  rm -f $O/$1.ncu-rep
}
timeout 300 python tools/prof_kernels.py step 1024 single double quad 50 10 4 > $O/pk_step1024.log 2>&1
timeout 300 python tools/prof_kernels.py op 16384 half single double > $O/pk_op16384.log 2>&1
timeout 300 python tools/prof_kernels.py op 8192 single double quad > $O/pk_op8192.log 2>&1
timeout 300 python tools/prof_kernels.py lu 16384 half single double tensor > $O/pk_lu_tensor.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_step -c 1 -o $O/ncu_step1024 -f \
  python tools/prof_kernels.py step 1024 single double quad 50 10 4 > $O/ncu_step1024.log 2>&1; summ ncu_step1024
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_debug -c 2 -o $O/ncu_op16384 -f \
  python tools/prof_kernels.py op 16384 half single double > $O/ncu_op16384.log 2>&1; summ ncu_op16384
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_debug -c 2 -o $O/ncu_op8192 -f \
  python tools/prof_kernels.py op 8192 single double quad > $O/ncu_op8192.log 2>&1; summ ncu_op8192
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_batched -c 1 -o $O/ncu_batched -f \
  python tools/prof_kernels.py batched > $O/ncu_batched.log 2>&1; summ ncu_batched
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_lu_team -c 1 -o $O/ncu_lu_tensor -f \
  python tools/prof_kernels.py lu 16384 half single double tensor > $O/ncu_lu_tensor.log 2>&1; summ ncu_lu_tensor
timeout 1200 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kernels > $O/ncu_launches.log 2>&1
du -sh $O
