#!/bin/bash
# ext tests (all, no -x) + full gpu suite + bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ext.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_ext.log 2>&1
echo "ext exit $?" >> gpurun_out/pytest_ext.log
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 --durations=8 -p no:cacheprovider --deselect tests/test_gpu_ext.py > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
