# Large-volume prefetch kernel: memcheck / synccheck / racecheck on a >1024-tile
# volume stopped by max_iters, then the whole -m gpu suite, smoke and the bench.
cd $GRAFT_REPO_ROOT
for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py large_owner > gpurun_out/sanitizer_pf_$t.txt 2>&1
  echo "== $t"; grep -E "iters=|ERROR SUMMARY|RACECHECK SUMMARY|Race reported|Barrier error" gpurun_out/sanitizer_pf_$t.txt | sort | uniq -c | cut -c1-160
done
bash tools/gpu_check.sh
