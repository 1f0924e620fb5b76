# Same-box A/B incl. a 17 M-voxel volume (owner path, one rank of an 8-GPU C4).
cd $GRAFT_REPO_ROOT
A=$GRAFT_REPO_ROOT/paper_1601_00072_b200/libfcm_b200_base.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
for r in 1 2; do for v in A B; do
  if [ $v = A ]; then export FCM_B200_LIB=$A; else unset FCM_B200_LIB; fi
  for cfg in C4 C2; do
    timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 10 > gpurun_out/ab_${v}_${cfg}_$r.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_${cfg}_$r.json')); print('$v $cfg run$r', round(d['value']/1e9,2), 'G', round(d['ms_per_step'],4), 'ms')"
  done
  timeout 300 python tools/pass_phases.py C3@16777216 C3@1000000 C1 --warm 5 2>&1 | grep -E "^C" | sed "s/^/$v run$r /"
done; done
for v in A B; do
  if [ $v = A ]; then export FCM_B200_LIB=$A; else unset FCM_B200_LIB; fi
  timeout 600 python tools/rank_proxy.py 2>&1 | grep -E "^ 8 " | sed "s/^/$v rank8 /"
done
