# GPU round trip: tests, smoke, benches.  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 600 python bench.py --steps 30 --warmup 3 --kernel ldg --no-cpu-baseline > gpurun_out/bench_C4_ldg.json 2> gpurun_out/bench_C4_ldg.err
timeout 600 python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 1200 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in gpurun_out/bench_C*.json; do echo $f; python -c "
import json; d=json.load(open('$f'))
print(round(d['value']/1e9,2), 'Gvox-it/s; pass_ms', d['pass_ms'], 'pro_ms', d.get('prologue_ms'), 'frac', d['roofline']['frac'], 'e2e', round(d['e2e']['value']/1e9,2), d['clocks'], d['plan'], d.get('cpu_baseline'))" ; done
cat gpurun_out/bench_ref.json
for f in gpurun_out/bench_*.err; do tail -n 3 $f; done
