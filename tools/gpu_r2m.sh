#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02c
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
PHASES=1 timeout 900 python tools/run_config.py cfg5 --max-cycles 3 > $O/cfg5_c3.log 2>&1
echo "rc=$?" >> $O/cfg5_c3.log; tail -n 24 $O/cfg5_c3.log
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_solve.py -m gpu -q -x -k "config5 or config1 or wellposed or config2 or table6" > $O/pytest_sub.log 2>&1
tail -n 4 $O/pytest_sub.log
timeout 300 python tools/prof_kernels.py step 16384 half single double 200 30 2 > $O/pk_step16384.log 2>&1 &&
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:k_step -c 1 -o $O/ncu_step16384 -f \
  python tools/prof_kernels.py step 16384 half single double 200 30 2 > $O/ncu_step16384.log 2>&1
$NCU -i $O/ncu_step16384.ncu-rep --page details --csv > $O/ncu_step16384_details.csv 2>&1
$NCU -i $O/ncu_step16384.ncu-rep --page raw --csv > $O/ncu_step16384_raw.csv 2>&1
gzip -f $O/ncu_step16384_raw.csv; rm -f $O/ncu_step16384.ncu-rep
cat $O/pk_step16384.log
