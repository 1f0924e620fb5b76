# compute-sanitizer over tools/sanitize.py (C1 solves in every launch mode).
cd $GRAFT_REPO_ROOT
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|iters=|Error|error" gpurun_out/sanitizer_$tool.txt | head -20
done
