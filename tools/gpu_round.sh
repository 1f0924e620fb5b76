# Round check on one B200: GPU tests, smoke, default bench (C4 + cpu_baseline),
# reference arm, and the ncu launch list of the default bench command.
# Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/launches_C4.err
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -3
cat gpurun_out/bench_C4.json; tail -3 gpurun_out/bench_C4.err
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
wc -l gpurun_out/launches_C4.csv; tail -2 gpurun_out/launches_C4.err
