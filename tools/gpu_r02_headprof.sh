#!/bin/bash
# HEAD capture: ncu --set full (with source) of the block kernel for configs 3, 2, 4, then the default bench.
mkdir -p gpurun_out/head
O=gpurun_out/head
for c in 3 2 4; do
  PROF_CONFIG=$c PROF_FRAMES=120 PROF_REPS=3 timeout 600 python tools/prof_run.py > $O/prof_plain_cfg$c.log 2>&1 && \
  PROF_CONFIG=$c PROF_FRAMES=120 PROF_REPS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 1 \
    -o $O/head_cfg$c -f python tools/prof_run.py > $O/ncu_cfg$c.log 2>&1
  echo "cfg $c rc=$?" >> $O/ncu_cfg$c.log
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
ls -la $O
