# Iteration: targeted GPU tests, bench C2/C4, pass phases, exchange latency on one GPU.
cd $GRAFT_REPO_ROOT
SEL=${PYTEST_SEL:-"tests/test_gpu_ops.py tests/test_gpu_parity.py"}
timeout 1200 python -m pytest $SEL -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 300 python tools/pass_phases.py C1 C3@1000000 C2 > gpurun_out/pass_phases.txt 2>&1
timeout 600 python tools/exchange_latency.py C2 > gpurun_out/exchange_C2.txt 2>&1
timeout 600 python tools/exchange_latency.py C4 > gpurun_out/exchange_C4.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log
for f in C2 C4; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d['value']/1e9, 'G', d['ms_per_step'], 'ms', d['roofline']['frac'], d.get('clocks'), 'recomp', (d.get('effective_recompute') or {}).get('value'))" ; tail -2 gpurun_out/bench_$f.err; done
grep -E "^C|solve|next" gpurun_out/pass_phases.txt
cat gpurun_out/exchange_C2.txt gpurun_out/exchange_C4.txt
