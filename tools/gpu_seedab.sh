cd $GRAFT_REPO_ROOT
for spec in "" "--no-seed-pass" "" "--no-seed-pass"; do
  timeout 600 python bench.py $spec --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('${spec:-seedpass}', round(d['value']/1e9,1), 'ms/step', round(d['ms_per_step'],3), 'pass_ms', round(d['pass_ms'],4), 'pro', round(d['prologue_ms'],3), 'loop', round(d['loop_kernel_ms'],3), d['clocks'])" || tail -3 gpurun_out/ab.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prologue -s 3 -c 1 \
   -o gpurun_out/prof_pro2_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-seed-pass > /dev/null 2>&1
