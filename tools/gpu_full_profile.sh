#!/bin/bash
# Full measurement pass for profiles/: tests, smoke, bench, config sweep, launch list, ncu --set full of
# the block kernel for configs 3, 2, 4 (each after its own plain run exited 0).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python tools/config_sweep.py > gpurun_out/sweep.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused_kernel|finalize_kernel|generic" -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
for c in 3 2 4; do
  PROF_CONFIG=$c PROF_FRAMES=120 PROF_REPS=3 timeout 600 python tools/prof_run.py > gpurun_out/prof_plain_cfg$c.log 2>&1 && \
  PROF_CONFIG=$c PROF_FRAMES=120 PROF_REPS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 1 \
    -o gpurun_out/prof_cfg$c -f python tools/prof_run.py > gpurun_out/ncu_cfg$c.log 2>&1
done
for f in gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log; do echo "== $f"; tail -n 2 "$f" | cut -c1-300; done
