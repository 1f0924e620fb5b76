# Evidence for the current default path: GPU tests, smoke, bench lines (C4 default, C2, C5), reference arm,
# launch list of the default bench command, ncu --set full of the loop kernel (C4, C2, C5s) and the prologue.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/launches_C4.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C5s python bench.py --config C5s --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C5s.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -1
for f in C4 C2 C5; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json'))
print('$f', round(d['value']/1e9,1), 'G; ms/step', round(d['ms_per_step'],3), 'pass', round(d['pass_ms'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), d['clocks'])"; done
cut -c1-200 gpurun_out/bench_ref.json
for f in gpurun_out/ncu_*.log; do tail -n 1 $f; done
