mkdir -p gpurun_out
./tools/micro/pipes > gpurun_out/micro_pipes.txt 2>&1
for c in 2 4; do
PROF_CONFIG=$c PROF_FRAMES=120 PROF_REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 1 \
  -o gpurun_out/prof_cfg$c -f python tools/prof_run.py > gpurun_out/ncu_cfg$c.log 2>&1
done
cat gpurun_out/micro_pipes.txt
