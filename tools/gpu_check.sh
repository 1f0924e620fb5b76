# One B200 check: selected GPU tests (PYTEST_SEL, default the whole -m gpu suite), smoke,
# default bench line (C4, cpu_baseline, e2e_api), the reference arm.  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
SEL=${PYTEST_SEL:-tests}
timeout 1500 python -m pytest $SEL -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
tail -15 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
python - <<'PY'
import json
for f in ("bench_C4", "bench_ref"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
    except Exception as e:
        print(f, "missing", e); continue
    keys = ("value", "ms_per_step", "e2e", "e2e_api", "cpu_baseline", "roofline", "clocks")
    print(f, json.dumps({k: d.get(k) for k in keys})[:3000])
PY
