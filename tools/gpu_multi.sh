#!/bin/bash
# exercise the torchrun (N>1) plumbing on a 1-GPU box with gloo, then the bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-e2e > gpurun_out/multi.log 2>&1
echo "multi exit $?" >> gpurun_out/multi.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.log 2>&1
echo "ref exit $?" >> gpurun_out/ref.log
