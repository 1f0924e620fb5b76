# Iteration: targeted GPU tests, bench C2/C4 (x2 each), pass phases, sanitizers on the C1 launch modes.
cd $GRAFT_REPO_ROOT
SEL=${PYTEST_SEL:-"tests/test_gpu_ops.py tests/test_gpu_parity.py tests/test_gpu_boundary.py"}
timeout 1200 python -m pytest $SEL -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for r in 1 2; do
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2_$r.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_C4_$r.json 2> gpurun_out/bench_C4.err
done
timeout 300 python tools/pass_phases.py C1 C3@1000000 C2 > gpurun_out/pass_phases.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log
for f in C2_1 C4_1 C2_2 C4_2; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d['value']/1e9, 'G', d['ms_per_step'], 'ms', d['roofline']['frac'], d.get('clocks'))" ; done
grep -E "^C|solve|next" gpurun_out/pass_phases.txt
if [ -n "$SAN" ]; then bash tools/gpu_sanitize.sh; fi
if [ -n "$E2E" ]; then timeout 900 python tools/e2e_phases.py > gpurun_out/e2e_phases.txt 2>&1; cat gpurun_out/e2e_phases.txt; fi
