cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b_C4.json 2> gpurun_out/b_C4.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_C5_lut.json 2> gpurun_out/b_C5_lut.err
timeout 600 python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b_C2.json 2> gpurun_out/b_C2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass_tma -s 3 -c 1 \
   -o gpurun_out/prof_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass_tma -s 3 -c 1 \
   -o gpurun_out/prof_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_C4.log 2>&1
for f in gpurun_out/b_*.json; do echo $f; python -c "
import json; d=json.load(open('$f'))
print(round(d['value']/1e9,2), 'Gvox-it/s; ms/step', round(d['ms_per_step'],3), 'pass_ms', round(d['pass_ms'],4), 'pro_ms', round(d.get('prologue_ms'),3), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), 'launches', d['gpu_launches'], d['clocks'])" ; done
for f in gpurun_out/b_*.err gpurun_out/ncu_*.log; do tail -n 2 $f; done
