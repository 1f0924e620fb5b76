# Full GPU suite + smoke + exchange latency + bench C2/C4.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python tools/exchange_latency.py C2 > gpurun_out/exchange_C2.txt 2>&1
timeout 600 python tools/exchange_latency.py C4 > gpurun_out/exchange_C4.txt 2>&1
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
tail -3 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head; tail -1 gpurun_out/smoke.log
for f in C2 C4; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d['value']/1e9, 'G', d['ms_per_step'], 'ms', d['roofline']['frac'], d.get('clocks'))" ; tail -2 gpurun_out/bench_$f.err; done
cat gpurun_out/exchange_C2.txt gpurun_out/exchange_C4.txt
