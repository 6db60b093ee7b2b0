#!/bin/bash
# Final round evidence: full GPU session (tests, smoke, bench, 2-rank, reference arm),
# launch list + ncu captures, every BASELINE config.
cd "$(dirname "$0")/.."
TAG=${1:-r02q}
bash tools/gpu_round.sh $TAG
bash tools/gpu_cfgs.sh "PM_BWD_WIDE=1" 130m 1.4b 2.8b 2.8b-16k
