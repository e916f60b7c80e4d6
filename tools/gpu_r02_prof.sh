#!/bin/bash
# tcgen05 probe + ncu --set full (with source) of the block kernel for configs 3, 2, 4 at HEAD.
mkdir -p gpurun_out
git_rev=$(cat .git_rev 2>/dev/null)
timeout 300 ./tools/micro/tc05 > gpurun_out/tc05.txt 2>&1; echo "tc05 rc=$?" >> gpurun_out/tc05.txt
for c in 3 2 4; do
  PROF_CONFIG=$c PROF_FRAMES=120 PROF_REPS=3 timeout 600 python tools/prof_run.py > gpurun_out/prof_plain_cfg$c.log 2>&1 && \
  PROF_CONFIG=$c PROF_FRAMES=120 PROF_REPS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 1 \
    -o gpurun_out/r02_cfg$c -f python tools/prof_run.py > gpurun_out/ncu_cfg$c.log 2>&1
  echo "cfg $c rc=$?" >> gpurun_out/ncu_cfg$c.log
done
ls -la gpurun_out/*.ncu-rep
cat gpurun_out/tc05.txt
