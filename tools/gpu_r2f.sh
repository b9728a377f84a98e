#!/bin/bash
# round-2: hunt the k_step fault at G = 148, pair-kernel epilogue
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
(cd tools/micro && for a in "16384 1024 1" "16384 2048 1" "8192 1024 1"; do timeout -k 10 90 ./tcgemm $a; echo "rc=$?"; done) > gpurun_out/tcgemm3.log 2>&1
cat gpurun_out/tcgemm3.log
for n in 8192 9472; do
timeout 600 python tools/run_config.py cfg5 --n $n --max-cycles 2 > gpurun_out/cfg5_$n.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_$n.log
tail -n 5 gpurun_out/cfg5_$n.log
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 8 python tools/run_config.py cfg5 --n 9472 --max-cycles 2 > gpurun_out/cfg5_san.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_san.log
grep -v "^$" gpurun_out/cfg5_san.log | head -n 60
