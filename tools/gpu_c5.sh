# C5 (c=8, m=1.5, 536M voxels) loop vs per-pass, plus C5s timeline, after GPU tests.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for spec in "" "--no-loop"; do
  timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline $spec > gpurun_out/c5.json 2>gpurun_out/c5.err
  python -c "
import json; d=json.load(open('gpurun_out/c5.json'))
print('C5 ${spec:-loop}', round(d['value']/1e9,1), 'ms/step', round(d['ms_per_step'],1), 'pass_ms', round(d['pass_ms'],3), 'per-pass', round(d['per_pass_launch_ms'],3), 'frac', round(d['roofline']['frac'],3), 'iters', d['config']['iterations_per_solve'], d['clocks'])" || tail -3 gpurun_out/c5.err
done
