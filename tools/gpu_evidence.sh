#!/bin/bash
# Round evidence in one call: full GPU session + launch list + ncu captures
# (gpu_round.sh), every BASELINE config, compute-sanitizer runs.
cd "$(dirname "$0")/.."
TAG=${1:-r02m}
bash tools/gpu_round.sh $TAG
bash tools/gpu_cfgs.sh "PM_BWD_WIDE=1" 130m 1.4b 2.8b 2.8b-16k
bash tools/gpu_sanitize.sh
