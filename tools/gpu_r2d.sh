#!/bin/bash
# round-2: CTA-pair tcgen05 update micro, cfg5 phase breakdown
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
(cd tools/micro && for a in "4096 256 1" "16384 256 1" "16384 512 1" "16384 1024 1" "16384 1024 0" "16384 2048 1"; do timeout -k 10 90 ./tcgemm $a; echo "rc=$?"; done) > gpurun_out/tcgemm2.log 2>&1
cat gpurun_out/tcgemm2.log
PHASES=1 timeout 600 python tools/run_config.py cfg5 --n 4096 --max-cycles 2 > gpurun_out/cfg5_4096_ph.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_4096_ph.log
tail -n 25 gpurun_out/cfg5_4096_ph.log
PHASES=1 timeout 1200 python tools/run_config.py cfg5 --max-cycles 3 > gpurun_out/cfg5_c3.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_c3.log
tail -n 25 gpurun_out/cfg5_c3.log
