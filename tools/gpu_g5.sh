cd $GRAFT_REPO_ROOT
bash tools/gpu_dev.sh "tests/test_gpu_parity.py" "PM_BWD_WIDE=0" libpm_a82.so libpm_a81.so libpm_a41.so
bash tools/gpu_ncu_w.sh r02f_a82 scan_bwd_wide PM_LIB=$PWD/paper_2408_03865_b200/libpm_a82.so
