# Same-box A/B of two library builds: A = paper_1601_00072_b200/libfcm_b200_base.so, B = the default build.
# Interleaved bench runs (C2, C4, C1 phases) so box-to-box variance cancels.
cd $GRAFT_REPO_ROOT
A=$GRAFT_REPO_ROOT/paper_1601_00072_b200/libfcm_b200_base.so
SEL=${PYTEST_SEL:-"tests/test_gpu_parity.py tests/test_gpu_ops.py"}
timeout 1200 python -m pytest $SEL -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for r in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then export FCM_B200_LIB=$A; else unset FCM_B200_LIB; fi
    for cfg in C2 C4; do
      timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 10 > gpurun_out/ab_${v}_${cfg}_$r.json 2>/dev/null
      python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_${cfg}_$r.json')); print('$v $cfg run$r', round(d['value']/1e9,2), 'G', round(d['ms_per_step'],4), 'ms', d.get('clocks',{}).get('sm_mhz'))"
    done
  done
done
unset FCM_B200_LIB
timeout 300 python tools/pass_phases.py C1 C3@1000000 C2 2>&1 | grep -E "^C"
FCM_B200_LIB=$A timeout 300 python tools/pass_phases.py C1 C3@1000000 C2 2>&1 | grep -E "^C" | sed 's/^/A: /'
