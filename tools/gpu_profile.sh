# Bench + ncu evidence for the pass kernel (one GPU).  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
CFG=${CFG:-C4}
timeout 900 python bench.py --config $CFG --steps 30 --warmup 3 > gpurun_out/bench_${CFG}.json 2> gpurun_out/bench_${CFG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
   --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pass_tma -s 30 -c 1 \
   -o gpurun_out/prof_pass_${CFG} python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${CFG}.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:prologue -s 1 -c 1 \
   -o gpurun_out/prof_prologue_${CFG} python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pro_${CFG}.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_${CFG}.json')); print({k: d[k] for k in ('value','pass_ms','prologue_ms','ms_per_step','clocks','cpu_baseline') if k in d}, d['roofline']['frac'], d['e2e'])"
tail -3 gpurun_out/ncu_full_${CFG}.log; ls -la gpurun_out/
