# synccheck over the cases it can instrument (per_pass_graph excluded: see profiles/sanitizer_r02.md),
# then the C4 launch list and ncu --set full of the (prefetching) loop kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py loop_kernel loop_kernel_m15_lut \
   per_pass_host prologue_kernel recompute shards4 u16 f64 c20 large_owner > gpurun_out/sanitizer/sanitizer_synccheck.txt 2>&1
grep -E "iters=|ERROR SUMMARY" gpurun_out/sanitizer/sanitizer_synccheck.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/launches_C4.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:loop_tma -s 3 -c 1 \
   -o gpurun_out/prof_loop_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_C4.log 2>&1
tail -n 2 gpurun_out/ncu_loop_C4.log
