#!/bin/bash
# round-2 evidence run: full GPU suite, cfg5 bench (both arms), ncu captures
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=12 > $O/pytest_gpu.log 2>&1
echo "rc=$?" >> $O/pytest_gpu.log
tail -n 6 $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
echo "bench rc=$?"; tail -n 12 $O/bench_cfg5.err; cut -c1-1500 $O/bench_cfg5.json
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg5.json 2> $O/bench_ref_cfg5.err
echo "ref rc=$?"; cut -c1-1200 $O/bench_ref_cfg5.json
summ() {
  $NCU -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>&1
  $NCU -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>&1
  gzip -f $O/$1_raw.csv
  rm -f $O/$1.ncu-rep
}
timeout 300 python tools/prof_kernels.py op 16384 half single double > $O/pk_op16384.log 2>&1 &&
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_debug -c 2 -o $O/ncu_op16384 -f \
  python tools/prof_kernels.py op 16384 half single double > $O/ncu_op16384.log 2>&1; summ ncu_op16384
timeout 300 python tools/prof_kernels.py lu 16384 half single double tensor > $O/pk_lu_tensor.log 2>&1 &&
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tc_update2 -s 60 -c 2 -o $O/ncu_tc_update -f \
  python tools/prof_kernels.py lu 16384 half single double tensor > $O/ncu_tc_update.log 2>&1; summ ncu_tc_update
cat $O/pk_op16384.log $O/pk_lu_tensor.log
du -sh $O
