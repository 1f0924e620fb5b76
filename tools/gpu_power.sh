# Steady-state comparison: loop kernel vs per-pass launches at C4 (long runs), timeline after a warm period.
cd $GRAFT_REPO_ROOT
for mode in "" "--no-loop" "" "--no-loop"; do
  timeout 600 python bench.py --steps 80 --warmup 10 --no-cpu-baseline $mode > gpurun_out/p.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/p.json'))
print('${mode:-loop}', 'ms/step', round(d['ms_per_step'],3), 'pass_ms', round(d['pass_ms'],4), d['clocks'])"
done
python tools/loop_timeline.py --config C4 --warm 60 > gpurun_out/tl_C4w.txt 2>&1; head -6 gpurun_out/tl_C4w.txt; tail -3 gpurun_out/tl_C4w.txt
