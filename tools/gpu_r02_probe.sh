cd $GRAFT_REPO_ROOT
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize.py > gpurun_out/sanitizer_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/sanitizer_synccheck.txt
for m in sync mbar tma; do timeout 120 compute-sanitizer --tool racecheck tools/racecheck_control/mbar_control $m > gpurun_out/racecheck_control_$m.txt 2>&1; echo "control $m rc=$?"; grep -E "mode|RACECHECK SUMMARY|Error" gpurun_out/racecheck_control_$m.txt | head -5; done
timeout 600 python tools/pass_phases.py C1 C3@1000000 C2 2>&1 | tee gpurun_out/pass_phases.txt
