#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02b
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 600 python tools/op_check.py > $O/op_check.log 2>&1; cat $O/op_check.log
PHASES=1 timeout 600 python tools/run_config.py cfg5 --n 4096 --max-cycles 2 > $O/cfg5_4096_ph.log 2>&1
echo "rc=$?" >> $O/cfg5_4096_ph.log; tail -n 22 $O/cfg5_4096_ph.log
timeout 600 python tools/crash_hunt.py > $O/crash_hunt.log 2>&1; cut -c1-400 $O/crash_hunt.log
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
echo "rc=$?" >> $O/pytest_gpu.log; tail -n 6 $O/pytest_gpu.log
summ() {
  $NCU -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>&1
  $NCU -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>&1
  gzip -f $O/$1_raw.csv
  rm -f $O/$1.ncu-rep
}
timeout 300 python tools/prof_kernels.py lu 16384 half single double tensor > $O/pk_lu_tensor.log 2>&1 &&
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tc_update2 -s 31 -c 1 -o $O/ncu_tc_update -f \
  python tools/prof_kernels.py lu 16384 half single double tensor > $O/ncu_tc_update.log 2>&1; summ ncu_tc_update
