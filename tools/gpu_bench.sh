#!/bin/bash
# bench only (+ optional env), 2 repeats
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/bench_$i.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$i.log
done
