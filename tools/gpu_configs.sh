#!/bin/bash
# bench every BASELINE config once (no cpu baseline / e2e), JSON lines -> gpurun_out/configs.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/configs.log
for c in 130m 1.4b 2.8b 2.8b-16k; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 >> gpurun_out/configs.log
done
