#!/bin/bash
# Round-2 measurement pass: smoke, GPU tests, default bench, sustained bench (power cap), the ncu
# launch list of the bench command, and the family sweep for the other configs.
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --steps 1000 --no-cpu --no-e2e --no-config5 > $O/bench_k1000_sustained.json 2>&1
timeout 600 python tools/config_sweep.py > $O/config_sweep.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused_kernel|finalize_kernel|generic" -c 400 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-config5 > $O/ncu_launch.log 2>&1
for n in 2 4; do
  VCA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus $n --steps 3 --warmup 3 --no-e2e --verify > $O/bench_gloo_n$n.log 2>&1
  echo "gloo n=$n rc=$?" >> $O/bench_gloo_n$n.log
done
for f in $O/smoke.log $O/pytest_gpu.log $O/bench.err; do echo "== $f"; tail -n 3 "$f" | cut -c1-300; done
