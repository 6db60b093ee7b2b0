#!/bin/bash
# ncu evidence: launch list (time per launch) + full-set capture of the scan kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-prof}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'(scan|conv|seg|pack)_' -c 60 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_ -s 8 -c 2 \
   -o gpurun_out/${TAG}_scan python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_ -s 8 -c 3 \
   -o gpurun_out/${TAG}_conv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_conv.log 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
tail -c 1500 gpurun_out/bench.log
ls -la gpurun_out
