#!/bin/bash
# Full GPU session: build, pytest -m gpu, smoke, bench (N=1), the torchrun
# 2-rank plumbing run (gloo on one GPU), the reference arm.  Logs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider -rA > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-e2e > gpurun_out/multi.log 2>&1
echo "multi exit $?" >> gpurun_out/multi.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.log 2>&1
echo "ref exit $?" >> gpurun_out/ref.log
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3
tail -2 gpurun_out/smoke.log gpurun_out/multi.log gpurun_out/ref.log
tail -c 1500 gpurun_out/bench.log
