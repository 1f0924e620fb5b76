"""Full-size parity at a BASELINE config: the GPU solve vs the reference's own
block-parallel engine (oracle/_ref, compiled Cython, all host threads) from
the same seeded start.  Measurement infrastructure (imports the reference).

    python tools/parity_full.py --config C4 [--out profiles/parity_C4_r01.json]

Checks the north-star bars: same iteration count and converged flag, centers
within 1e-4 relative, memberships within 1e-5 absolute, labels identical
(mismatches listed with their membership margins), objective trace.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
import bench  # noqa: E402
import fcmseg  # noqa: E402
from fcmseg import core, parallel  # noqa: E402

import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--out", default=None)
args = ap.parse_args()
shape, c, m, eps = bench.CONFIGS[args.config]
x8 = bench.make_volume(shape)
n = x8.shape[0]

t0 = time.perf_counter()
with pkg.FcmPlan(n, c, _lib.FCM_X_U8) as plan:
    plan.upload_pixels(x8)
    plan.init_membership(0)
    v, trace, k, conv = plan.run(m, eps, 500)
    u, lab = plan.download()
t_gpu = time.perf_counter() - t0

x = x8.astype(np.float64)
cfg = fcmseg.FcmConfig(c=c, m=m, epsilon=eps, max_iters=500, seed=0)
u0 = core.init_membership(n, cfg).u
del x8
workers = os.cpu_count() or 1
t0 = time.perf_counter()
rv, ru, rk, rtrace, rconv, _ = parallel._iterate(x, u0, cfg, workers)
t_ref = time.perf_counter() - t0
del u0
rlab = ru.reshape(n, c).argmax(axis=1).astype(np.int32)

du = np.abs(u - ru)
mism = np.nonzero(lab != rlab)[0]
out = {
    "config": args.config, "n_voxels": int(n), "c": c, "m": m, "epsilon": eps,
    "iterations": {"gpu": int(k), "reference": int(rk)},
    "converged": {"gpu": bool(conv), "reference": bool(rconv)},
    "centers_gpu": [float(t) for t in v], "centers_reference": [float(t) for t in rv],
    "centers_max_rel": float(np.max(np.abs(v - rv) / np.abs(rv))),
    "membership_max_abs": float(du.max()),
    "label_mismatches": int(mism.size),
    "trace_max_rel": float(np.max(np.abs(np.array(trace) - np.array(rtrace)) / np.abs(np.array(rtrace)))),
    "gpu_solve_s_incl_download": t_gpu, "reference_parallel_s": t_ref, "reference_workers": workers,
}
if mism.size:
    rows = ru.reshape(n, c)[mism[:10]]
    srt = np.sort(rows, axis=1)
    out["label_mismatch_margins"] = [float(t) for t in (srt[:, -1] - srt[:, -2])]
out["pass"] = (k == rk and conv == rconv and out["centers_max_rel"] <= 1e-4 and out["membership_max_abs"] <= 1e-5)
print(json.dumps(out, indent=1))
if args.out:
    json.dump(out, open(args.out, "w"), indent=1)
