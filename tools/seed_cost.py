"""Cost of the seeded pass 0 inside the loop kernel, one GPU.

    python tools/seed_cost.py [--config C4]

Times the persistent loop kernel with max_iters = 1, 2, 3 (CUDA events inside
the library, fcm_last_timing); pass 0 ~= 2 t(1) - t(2).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=7)
args = ap.parse_args()
shape, c, m, eps = bench.CONFIGS[args.config]
x = bench.make_volume(shape)
plan = pkg.FcmPlan(x.shape[0], c, _lib.FCM_X_U8)
plan.upload_pixels(x)
res = {}
for k in (1, 2, 3):
    ts = []
    for _ in range(args.reps):
        plan.init_membership(0)
        plan.run(m, 1e-30, k)
        ts.append(plan.timing()["loop_ms"])
    res[k] = float(np.median(ts))
p0 = 2 * res[1] - res[2]
print(f"{args.config}: loop_ms t1 {res[1]:.4f} t2 {res[2]:.4f} t3 {res[3]:.4f} | pass {res[3]-res[2]:.4f} "
      f"{res[2]-res[1]:.4f} | seed pass0 ~ {p0:.4f} ms")
