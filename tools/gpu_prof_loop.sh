# ncu --set full of the loop kernel (C2, C4) and the per-pass kernel (C2).
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass_tma -s 20 -c 1 \
   -o gpurun_out/prof_pass_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline --no-loop > gpurun_out/ncu_pass_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C4.log 2>&1
for f in gpurun_out/ncu_*.log; do tail -n 2 $f; done
ls -la gpurun_out/*.ncu-rep
