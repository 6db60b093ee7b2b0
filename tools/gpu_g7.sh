cd $GRAFT_REPO_ROOT
bash tools/gpu_cfgs.sh "PM_BWD_WIDE=1|PM_BWD_WIDE=0" 130m 2.8b
bash tools/gpu_ncu_w.sh r02g_w41 scan_bwd_wide
