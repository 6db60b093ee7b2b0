cd $GRAFT_REPO_ROOT
bash tools/gpu_dev.sh "tests/test_gpu_parity.py" "PM_BWD_WIDE=1"
bash tools/gpu_ncu_w.sh r02j_convb conv_bwd_kernel
bash tools/gpu_ncu_w.sh r02j_convf conv_fwd_kernel
