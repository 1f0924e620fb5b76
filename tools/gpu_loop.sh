# Loop-kernel check: GPU tests, then C4/C2/C5 benches with and without the loop kernel.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
for cfg in C4 C2; do
  for mode in "" "--no-loop"; do
    tag=${cfg}${mode:+_noloop}
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline $mode > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
  done
done
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_C5.json 2> gpurun_out/b_C5.err
for f in gpurun_out/b_*.json; do echo $f; python -c "
import json; d=json.load(open('$f'))
print(round(d['value']/1e9,2), 'Gvox-it/s; ms/step', round(d['ms_per_step'],3), 'pass_ms', round(d['pass_ms'],4), 'per_pass_launch', round(d['per_pass_launch_ms'],4), 'pro_ms', round(d.get('prologue_ms'),3), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), 'launches', d['gpu_launches'], 'iters', d['config']['iterations_per_solve'], d['clocks'])" ; done
for f in gpurun_out/b_*.err; do tail -n 2 $f; done
