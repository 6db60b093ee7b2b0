#!/bin/bash
# ncu --set full of one kernel: bash tools/gpu_ncu_w.sh TAG REGEX [env...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=$1; RE=$2; shift 2
timeout 900 env "$@" ncu --set full --clock-control none --import-source on -k regex:"$RE" -s 2 -c 1 \
   -o gpurun_out/${TAG} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/${TAG}_ncu.log
