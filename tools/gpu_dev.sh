#!/bin/bash
# dev loop: build, targeted parity tests, bench A/B of env settings / library variants.
# usage: bash tools/gpu_dev.sh "TESTS" "ENV_A|ENV_B|..." [libvariant.so ...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest $1 -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_dev.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_dev.log
tail -3 gpurun_out/pytest_dev.log
IFS='|' read -ra ENVS <<< "$2"
shift 2
for i in 1 2; do
  for e in "${ENVS[@]}"; do
    tag=$(echo "$e" | tr -c 'A-Za-z0-9_' '_')
    timeout 300 env $e python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/dev_${tag}_$i.log 2>&1
  done
  for v in "$@"; do
    PM_LIB=$PWD/paper_2408_03865_b200/$v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/dev_lib_${v%.so}_$i.log 2>&1
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/dev_*.log")):
    ok = False
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); ok = True
            print(f[11:], round(d["ms_per_step"], 4), {k: round(v["ms"], 4) for k, v in d["kernels"].items()})
    if not ok:
        print(f, "FAILED:", open(f).read()[-800:])
PY
