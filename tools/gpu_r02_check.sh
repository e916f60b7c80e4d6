#!/bin/bash
# Round-2 check pass on one B200: GPU tests (parity, integer checks, mutation self-test), the
# default bench line, and the N > 1 bench path run functionally with gloo (ranks share the GPU).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,memory.total --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for n in 2 4; do
  VCA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus $n --steps 3 --warmup 3 --no-e2e --verify > gpurun_out/bench_gloo_n$n.log 2>&1
  echo "gloo n=$n rc=$?" >> gpurun_out/bench_gloo_n$n.log
done
for f in gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log gpurun_out/bench_gloo_n2.log gpurun_out/bench_gloo_n4.log; do echo "== $f"; tail -n 3 "$f" | cut -c1-400; done
