#!/bin/bash
# run an experiment script: bash tools/gpu_exp.sh script.py args...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python "$@" > gpurun_out/exp.log 2>&1
echo "exit $?" >> gpurun_out/exp.log
