# Same-box A/B (A = libfcm_b200_base.so, B = default build) at large volumes + C2, with phases.
cd $GRAFT_REPO_ROOT
A=$GRAFT_REPO_ROOT/paper_1601_00072_b200/libfcm_b200_base.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_headline.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
for r in 1 2; do
  for v in A B; do
    if [ $v = A ]; then export FCM_B200_LIB=$A; else unset FCM_B200_LIB; fi
    for cfg in C4 C2; do
      timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 10 > gpurun_out/ab_${v}_${cfg}_$r.json 2>/dev/null
      python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_${cfg}_$r.json')); print('$v $cfg run$r', round(d['value']/1e9,2), 'G', round(d['ms_per_step'],4), 'ms', d.get('clocks',{}).get('sm_mhz'))"
    done
  done
done
unset FCM_B200_LIB
timeout 600 python tools/pass_phases.py C3@16777216 C4 --warm 5 2>&1 | grep -E "^C|barrier out|upper|next pass|consumers done"
FCM_B200_LIB=$A timeout 600 python tools/pass_phases.py C3@16777216 --warm 5 2>&1 | grep -E "^C|next pass" | sed 's/^/A: /'
timeout 600 python tools/exchange_latency.py C4 2>&1 | tail -5
