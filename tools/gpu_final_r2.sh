# Round-2 final evidence: the four compute-sanitizer tools over every tools/sanitize.py case
# (the large-volume prefetching loop kernel included), then tools/gpu_check.sh.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
CASES="loop_kernel loop_kernel_m15_lut per_pass_graph per_pass_host prologue_kernel recompute shards4 u16 f64 c20 large_owner"
for t in memcheck initcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py $CASES > gpurun_out/sanitizer/sanitizer_$t.txt 2>&1
  echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitizer/sanitizer_$t.txt
  grep -c "iters=" gpurun_out/sanitizer/sanitizer_$t.txt
  grep -E "Write access at|Error: " gpurun_out/sanitizer/sanitizer_$t.txt | sed 's/(const.*)+/+/' | cut -c1-140 | sort | uniq -c | head -8
done
bash tools/gpu_check.sh
