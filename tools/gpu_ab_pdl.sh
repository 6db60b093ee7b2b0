#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_main_$i.log 2>&1
  PM_NO_PDL=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_nopdl_$i.log 2>&1

done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f, round(d["ms_per_step"], 4), d.get("overlap", {}).get("scan_fwd_bwd_ms"), {k: round(v["ms"], 4) for k, v in d["kernels"].items()})
PY
