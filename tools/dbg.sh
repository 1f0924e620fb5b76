cd $GRAFT_REPO_ROOT
for args in "200003 16 2.0 0" "200003 16 2.0 1" "200003 8 2.0 1" "200003 3 2.0 1" "7109137 3 2.0 1" "200003 16 2.0 0 3" "5000000 16 2.0 1"; do
  echo "== $args"; timeout 60 python tools/debug_case.py $args 2>&1 | tail -3
done
python tools/loop_timeline.py --config C4 > gpurun_out/tl_C4.txt 2>&1; head -5 gpurun_out/tl_C4.txt; tail -4 gpurun_out/tl_C4.txt
python tools/loop_timeline.py --config C2 > gpurun_out/tl_C2.txt 2>&1; head -5 gpurun_out/tl_C2.txt; tail -4 gpurun_out/tl_C2.txt
