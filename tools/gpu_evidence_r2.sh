# Round-2 evidence on one B200: full GPU suite (headline parity records into gpurun_out/parity),
# smoke, sanitizers, default bench line (+ reference arm), C2 / C5 bench lines, pass phases,
# exchange latency, launch list and ncu --set full of the loop kernel at C4 and C2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/parity
FCM_PARITY_LOG=gpurun_out/parity timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
if [ -n "$SAN" ]; then bash tools/gpu_sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1; fi
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 900 python bench.py --config C5 --no-cpu-baseline --steps 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 600 python tools/pass_phases.py C1 C3@1000000 C2 C3@16777216 > gpurun_out/pass_phases.txt 2>&1
timeout 600 python tools/exchange_latency.py C2 > gpurun_out/exchange_C2.txt 2>&1
timeout 600 python tools/exchange_latency.py C4 > gpurun_out/exchange_C4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/launches_C4.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C2.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head; tail -1 gpurun_out/smoke.log
grep -E "^==|ERROR SUMMARY|Race reported" gpurun_out/sanitize_summary.txt | sort | uniq -c | head -20
for f in C4 C2 C5 ref; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), d.get('clocks'), (d.get('e2e') or {}).get('value'))" ; tail -1 gpurun_out/bench_$f.err; done
grep -E "^C|solve|next" gpurun_out/pass_phases.txt
cat gpurun_out/exchange_C2.txt gpurun_out/exchange_C4.txt
ls gpurun_out/parity
timeout 600 python tools/rank_proxy.py --exchange-us 2.4,2.3,3.5 > gpurun_out/rank_proxy.txt 2>&1; tail -9 gpurun_out/rank_proxy.txt
timeout 900 python tools/e2e_phases.py > gpurun_out/e2e_phases.txt 2>&1; tail -10 gpurun_out/e2e_phases.txt
