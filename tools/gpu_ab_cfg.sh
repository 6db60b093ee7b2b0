#!/bin/bash
# A/B of library variants over configs: bash tools/gpu_ab_cfg.sh "130m 1.4b" libpm_b.so ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
CFGS=$1; shift
for c in $CFGS; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abc_main_$c.log 2>&1
  for v in "$@"; do
    PM_LIB=$PWD/paper_2408_03865_b200/$v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abc_${v%.so}_$c.log 2>&1
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/abc_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f, round(d["ms_per_step"], 4), round(d["overlap"]["serial_step_ms"], 4), {k: round(v["ms"], 4) for k, v in d["kernels"].items()})
PY
