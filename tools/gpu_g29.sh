cd $GRAFT_REPO_ROOT
bash tools/gpu_dev.sh "tests/test_gpu_parity.py tests/test_gpu_ext.py" "PM_BWD_WIDE=1" libpm_tp0.so
for c in 130m; do for v in "" "PM_LIB=$PWD/paper_2408_03865_b200/libpm_tp0.so"; do env $v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$c', '$v'[-12:], d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"; done; done
