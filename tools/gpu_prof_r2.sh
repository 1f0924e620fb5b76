# Round-2 evidence: launch list of the default bench, ncu --set full of the loop kernel at C4 and C2.
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/launches_C4.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C2.log 2>&1
for f in gpurun_out/ncu_*.log; do tail -n 2 $f; done
