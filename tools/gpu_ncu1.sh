#!/bin/bash
# one ncu --set full capture of one kernel (regex $1) in the bench step -> gpurun_out/$2.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$1" -s 4 -c 1 \
   -o gpurun_out/$2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu1.log
