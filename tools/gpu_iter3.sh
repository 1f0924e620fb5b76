# Iteration check: seed/LUT changes -- targeted GPU tests, bench C4 and C2, seed cost, ncu of the loop kernel at C4.
cd $GRAFT_REPO_ROOT
SEL=${PYTEST_SEL:-"tests/test_gpu_ops.py tests/test_gpu_parity.py"}
timeout 1200 python -m pytest $SEL -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 300 python tools/seed_cost.py > gpurun_out/seed_cost.txt 2>&1
if [ -n "$NCU" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C4.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log
for f in C2 C4; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d['value']/1e9, 'G', d['ms_per_step'], 'ms', d['roofline']['frac'], d.get('prologue_ms'), d.get('clocks'), 'recomp', (d.get('effective_recompute') or {}).get('value'))" ; tail -2 gpurun_out/bench_$f.err; done
cat gpurun_out/seed_cost.txt | tail -5
