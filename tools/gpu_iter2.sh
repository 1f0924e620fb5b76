# Iteration check on one B200: pass-phase timeline (C1, C3-1M, C2), C2 and C4 bench lines,
# then the bitwise/parity GPU tests named in PYTEST_SEL (default tests/test_gpu_parity.py).
cd $GRAFT_REPO_ROOT
timeout 300 python tools/pass_phases.py C1 C3@1000000 C2 > gpurun_out/pass_phases.txt 2>&1
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
SEL=${PYTEST_SEL:-tests/test_gpu_parity.py}
timeout 1200 python -m pytest $SEL -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
cat gpurun_out/pass_phases.txt
for f in C2 C4; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d['value']/1e9, 'G', d['ms_per_step'], 'ms', d['roofline']['frac'], d.get('clocks'))" ; tail -2 gpurun_out/bench_$f.err; done
tail -3 gpurun_out/pytest_gpu.log
