# racecheck control: the large-volume case with the HEAD library (no prefetch) vs the current one.
cd $GRAFT_REPO_ROOT
for v in A B; do
  if [ $v = A ]; then export FCM_B200_LIB=$GRAFT_REPO_ROOT/paper_1601_00072_b200/libfcm_b200_base.so; else unset FCM_B200_LIB; fi
  timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py large_owner > gpurun_out/sanitizer_rc_$v.txt 2>&1
  echo "== $v"; grep -E "iters=|RACECHECK SUMMARY" gpurun_out/sanitizer_rc_$v.txt
  grep -E "Write access at" gpurun_out/sanitizer_rc_$v.txt | sed 's/(const.*)+/+/' | cut -c1-140 | sort | uniq -c
done
