# Iteration check: GPU tests, loop-kernel timelines, benches (C4 loop/no-loop, C2, C5).
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for cfg in C2 C4; do python tools/loop_timeline.py --config $cfg > gpurun_out/tl_$cfg.txt 2>&1; head -6 gpurun_out/tl_$cfg.txt; done
for spec in "C4" "C4 --no-loop" "C2" "C2 --no-loop" "C5"; do
  set -- $spec; tag=$1${2:+_noloop}
  steps=20; [ $1 = C5 ] && steps=3
  timeout 900 python bench.py --config $1 $2 --steps $steps --warmup 3 --no-cpu-baseline > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/b_$tag.json'))
print('$tag', round(d['value']/1e9,2), 'Gvox-it/s; ms/step', round(d['ms_per_step'],3), 'pass_ms', round(d['pass_ms'],4), 'per_pass_launch', round(d['per_pass_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'iters', d['config']['iterations_per_solve'], d['clocks'])" || tail -3 gpurun_out/b_$tag.err
done
