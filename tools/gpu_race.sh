# racecheck on the loop-kernel cases of tools/sanitize.py, then the same-box A/B.
cd $GRAFT_REPO_ROOT
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py > gpurun_out/sanitizer_racecheck.txt 2>&1
grep -E "iters=|Race reported|RACECHECK SUMMARY" gpurun_out/sanitizer_racecheck.txt | cut -c1-150
bash tools/gpu_ab.sh
