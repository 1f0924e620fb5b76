# A/B of pass kernels (direct m2 product form vs intensity table) and loop modes, C4 and C2.
cd $GRAFT_REPO_ROOT
for cfg in C4 C2; do
  for k in tma lut; do
    for mode in "" "--no-loop"; do
      tag=${cfg}_${k}${mode:+_noloop}
      timeout 600 python bench.py --config $cfg --kernel $k --steps 20 --warmup 3 --no-cpu-baseline $mode > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
    done
  done
done
python tools/loop_timeline.py --config C2 --kernel 2 > gpurun_out/tl_C2_lut.txt 2>&1
for f in gpurun_out/ab_*.json; do echo $f; python -c "
import json; d=json.load(open('$f'))
print(round(d['value']/1e9,2), 'Gvox-it/s; ms/step', round(d['ms_per_step'],3), 'pass_ms', round(d['pass_ms'],4), 'per_pass_launch', round(d['per_pass_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), d['clocks'])" ; done
for f in gpurun_out/ab_*.err; do tail -n 2 $f; done
head -8 gpurun_out/tl_C2_lut.txt
