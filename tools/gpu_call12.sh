AB_STEPS=200 AB_CONFIGS="2" bash tools/gpu_ab.sh > /dev/null 2>&1
PROF_CONFIG=2 PROF_FRAMES=120 PROF_REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 1 -o gpurun_out/prof_cfg2 -f python tools/prof_run.py > gpurun_out/ncu_cfg2.log 2>&1
grep -E "===|round" gpurun_out/ab.log
