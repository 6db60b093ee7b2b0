#!/bin/bash
# ncu --set full (with source) of the scan fwd and bwd kernels in the bench step -> gpurun_out/$1_{fwd,bwd}.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for k in bwd fwd; do
  PM_NO_PDL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_${k}_kernel -s 4 -c 1 \
     -o gpurun_out/${TAG}_${k} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${k}.log 2>&1
done
ls gpurun_out
