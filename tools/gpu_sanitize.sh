#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck on the tiny
# and a small bf16 config, PDL forced on; 130m under memcheck.  Logs in
# gpurun_out/sanitize_*.log.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export PM_PDL=1
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in tiny small; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
      python tools/sanitize_run.py $cfg > gpurun_out/sanitize_${tool}_${cfg}.log 2>&1
    echo "exit $?" >> gpurun_out/sanitize_${tool}_${cfg}.log
  done
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py 130m \
  > gpurun_out/sanitize_memcheck_130m.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_memcheck_130m.log
tail -n 4 gpurun_out/sanitize_*.log
