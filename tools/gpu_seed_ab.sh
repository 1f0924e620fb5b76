# Same-box A/B: seeded start as the loop kernel's pass 0 (default) vs the separate prologue kernel.
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for cfg in C4 C2; do
    for v in loop pro; do
      if [ $v = pro ]; then X=--no-seed-pass; else X=; fi
      timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 10 $X > gpurun_out/sab_${v}_${cfg}_$r.json 2>/dev/null
      python -c "
import json; d=json.load(open('gpurun_out/sab_${v}_${cfg}_$r.json')); print('$v $cfg run$r', round(d['value']/1e9,2), 'G', round(d['ms_per_step'],4), 'ms', 'prologue_ms', round(d.get('prologue_ms') or 0,4))"
    done
  done
done
