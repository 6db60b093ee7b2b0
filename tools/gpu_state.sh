#!/bin/bash
# state check: parity tests + smoke + bench, then ncu source-level captures of both scans
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-state}
bash tools/gpu_quick.sh
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_bwd_kernel -s 4 -c 1 \
   -o gpurun_out/${TAG}_bwd python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_fwd_kernel -s 4 -c 1 \
   -o gpurun_out/${TAG}_fwd python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fwd.log 2>&1
ls gpurun_out
