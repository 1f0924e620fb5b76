# Round-2 baseline on one B200: GPU suite, smoke, bench C4/C2/C1, pass-phase timeline.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
for cfg in C2; do timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; done
timeout 300 python tools/pass_phases.py C1 C3@1000000 C2 > gpurun_out/pass_phases.txt 2>&1
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in C4 C2; do cut -c1-600 gpurun_out/bench_$f.json; tail -2 gpurun_out/bench_$f.err; done
cat gpurun_out/pass_phases.txt
