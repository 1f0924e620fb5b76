"""Paper Table-3-shaped sweep: GPU engine vs the reference's CPU engines.

    python tools/sweep_table3.py [--runs 3] [--out profiles/table3_r01]

SURVEY §8(d) configs C1 (181x217 slice) and C3 (C1 enlarged with the
reference's own `enlarge_dataset` to 40K..1M bytes, imgio.py:196-217), plus
C2 (181x217x181).  c=3, m=2, eps=1e-5, seed 0.  Rows follow the reference
harness (bench.py:22-23, CSV_HEADER: dataset_bytes,engine,run,seconds,
iterations) with a third engine, "gpu": one fcm_run on cuda:0 through the C
ABI (device seeded start + passes to convergence; CUDA events), and the two
reference engines timed exactly as bench._timed_loop does (bench.py:49-59)
from the same seeded start.  Iteration counts are asserted equal.  This is
measurement infrastructure: it imports the reference from oracle/_ref.
"""
import argparse
import csv
import json
import os
import statistics
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
import fcmseg  # noqa: E402  (the reference, built by oracle/build_ref.sh)
from fcmseg import core, parallel  # noqa: E402
from fcmseg.imgio import enlarge_dataset  # noqa: E402

import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from paper_1601_00072_b200.phantom import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--out", default=os.path.join(REPO, "profiles", "table3_r01"))
ap.add_argument("--cpu-max-pixels", type=int, default=1_300_000, help="skip the CPU engines above this size")
args = ap.parse_args()
assert fcmseg.backend_name() == "compiled"

c, m, eps = 3, 2.0, 1e-5
c1 = make_config("C1")
base = fcmseg.GrayImage(181, 217, c1.astype(np.float64))
datasets = [("C1", base)]
for label, target in (("40K", 40 * 1024), ("100K", 100 * 1024), ("200K", 200 * 1024), ("500K", 500 * 1024),
                      ("1M", 1024 * 1024)):
    datasets.append((f"C3-{label}", enlarge_dataset(base, target)))
c2 = make_config("C2")
datasets.append(("C2", fcmseg.GrayImage(181, 217 * 181, c2.astype(np.float64))))

workers = os.cpu_count() or 1
rows, summary = [], []
for name, img in datasets:
    x = np.asarray(img.pixels, dtype=np.float64)
    n = x.shape[0]
    cfg = fcmseg.FcmConfig(c=c, m=m, epsilon=eps, max_iters=500, seed=0)
    u0 = core.init_membership(n, cfg).u
    rec = {"dataset": name, "dataset_bytes": n}
    # --- GPU engine: uint8 pixels, device seeded start (bit-identical to u0)
    x8 = x.astype(np.uint8)
    assert np.array_equal(x8.astype(np.float64), x)
    with pkg.FcmPlan(n, c, _lib.FCM_X_U8) as plan:
        plan.upload_pixels(x8)
        plan.init_membership(0)
        for _ in range(3):
            plan.run(m, eps, 500)
        secs, iters = [], None
        for r in range(args.runs):
            _, _, k, conv = plan.run(m, eps, 500)
            t = plan.timing()
            secs.append(t["loop_ms"] / 1e3)
            iters = k
            rows.append((n, "gpu", r, repr(t["loop_ms"] / 1e3), k))
        rec["gpu"] = {"mean_s": statistics.fmean(secs), "iterations": iters,
                      "s_per_iter": statistics.fmean(secs) / iters,
                      "voxel_iter_per_s": n * iters / statistics.fmean(secs)}
    # --- reference engines (bench._timed_loop)
    if n <= args.cpu_max_pixels:
        for engine in ("sequential", "parallel"):
            secs = []
            for r in range(args.runs if n < 400_000 else 1):
                u = u0.copy()
                t0 = time.perf_counter()
                if engine == "sequential":
                    _, _, k, _, _ = core._iterate(x, u, cfg)
                else:
                    _, _, k, _, _, _ = parallel._iterate(x, u, cfg, workers)
                secs.append(time.perf_counter() - t0)
                rows.append((n, engine, r, repr(secs[-1]), k))
            assert k == iters, (name, engine, k, iters)
            rec[engine] = {"mean_s": statistics.fmean(secs), "iterations": k,
                           "s_per_iter": statistics.fmean(secs) / k,
                           "voxel_iter_per_s": n * k / statistics.fmean(secs)}
        rec["gpu_speedup_vs_sequential"] = rec["sequential"]["mean_s"] / rec["gpu"]["mean_s"]
        rec["gpu_speedup_vs_parallel"] = rec["parallel"]["mean_s"] / rec["gpu"]["mean_s"]
    summary.append(rec)
    print(json.dumps(rec), flush=True)

with open(args.out + ".csv", "w", newline="\n") as f:
    w = csv.writer(f, lineterminator="\n")
    w.writerow(("dataset_bytes", "engine", "run", "seconds", "iterations"))
    w.writerows(rows)
with open(args.out + ".json", "w") as f:
    json.dump({"host_threads": workers, "c": c, "m": m, "epsilon": eps, "rows": summary}, f, indent=1)
