# A/B: m=2 table (default) vs per-voxel product form (direct), loop vs per-pass, C4 + C2; steady-state.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for spec in "C4 tma" "C4 direct" "C4 tma --no-loop" "C4 direct --no-loop" "C2 tma" "C2 direct" "C4 tma" "C4 direct"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --kernel $2 $3 --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$spec', round(d['value']/1e9,1), 'Gvox-it/s ms/step', round(d['ms_per_step'],3), 'pass_ms', round(d['pass_ms'],4), 'frac', round(d['roofline']['frac'],3), d['clocks'])" || tail -3 gpurun_out/ab.err
done
python tools/loop_timeline.py --config C4 --warm 40 > gpurun_out/tl_C4w.txt 2>&1; head -5 gpurun_out/tl_C4w.txt
