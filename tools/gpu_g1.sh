cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/base_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_bwd_kernel -s 2 -c 1 -o gpurun_out/r02d_bwd python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02d_ncu.log 2>&1
echo done
