# Per-thread stage-empty arrivals: racecheck on the large volume, then the same-box A/B.
cd $GRAFT_REPO_ROOT
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py large_owner loop_kernel recompute > gpurun_out/sanitizer_rc_arrive.txt 2>&1
grep -E "iters=|RACECHECK SUMMARY" gpurun_out/sanitizer_rc_arrive.txt
grep -E "Write access at" gpurun_out/sanitizer_rc_arrive.txt | sed 's/(const.*)+/+/' | cut -c1-140 | sort | uniq -c | head
bash tools/gpu_ab_sizes.sh
