#!/bin/bash
# full session + ncu: bash tools/gpu_round.sh TAG
cd "$(dirname "$0")/.."
TAG=${1:-prof}
bash tools/gpu_full.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'(scan|conv|seg|pack)_' -c 60 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'scan_(fwd|bwd|bwd_wide)_kernel' -s 8 -c 2 \
   -o gpurun_out/${TAG}_scan python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_ -s 8 -c 3 \
   -o gpurun_out/${TAG}_conv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_conv.log 2>&1
ls gpurun_out
