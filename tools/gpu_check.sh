# GPU round trip: tests, smoke, bench (both pass kernels), launch list.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tma.json 2> gpurun_out/bench_tma.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --kernel ldg > gpurun_out/bench_ldg.json 2> gpurun_out/bench_ldg.err
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in gpurun_out/bench_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value']/1e9, 'Gvox-it/s pass_ms', d['pass_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value']/1e9, d['clocks'], d['plan'])" ; done
tail -3 gpurun_out/bench_*.err
