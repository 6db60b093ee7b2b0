#!/bin/bash
# occupancy sweep of the scan kernels (env tuning knobs), short benches
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/sweep.log
for cfg in "3 3" "4 4" "5 3" "6 4" "5 4" "4 3"; do
  set -- $cfg
  PM_TUNE_FWD_MINB=$1 PM_TUNE_BWD_MINB=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>&1
  python -c "
import json,sys
d=json.loads([l for l in open('gpurun_out/sw.json') if l.startswith('{')][0])
k=d['kernels']
print('fwd_minb=$1 bwd_minb=$2', 'step_ms=%.3f'%d['ms_per_step'], 'fwd=%.3f'%k['scan_fwd']['ms'], 'bwd=%.3f'%k['scan_bwd']['ms'])
" >> gpurun_out/sweep.log 2>&1
done
cat gpurun_out/sweep.log
