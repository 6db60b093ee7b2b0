#!/bin/bash
# bench every BASELINE config (+ env A/B): bash tools/gpu_cfgs.sh "ENV_A|ENV_B" cfg1 cfg2 ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
IFS='|' read -ra ENVS <<< "$1"; shift
for c in "$@"; do for e in "${ENVS[@]}"; do
  tag=$(echo "$c-$e" | tr -c 'A-Za-z0-9_.-' '_')
  timeout 600 env $e python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfgs/$tag.log 2>&1
done; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/cfgs/*.log")):
    ok = False
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); ok = True
            print(f.split("/")[-1], round(d["ms_per_step"], 4), {k: round(v["ms"], 4) for k, v in d["kernels"].items()})
    if not ok: print(f, "FAILED", open(f).read()[-600:])
PY
