"""Steady-state pass bandwidth of the loop kernel vs the number of clusters, one GPU.

    python tools/c_sweep.py [--shape 512 512 512] [--m 1.5 2.0]

Per (c, m): loop-kernel time at max_iters = 3 and 7 (no early stop); the
difference / 4 is one streaming pass; GB/s = n (1 + 8c) / pass (canonical
bytes).  Prints the ring depth the layout gives each c.
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
ap.add_argument("--shape", type=int, nargs=3, default=[512, 512, 512])
ap.add_argument("--m", type=float, nargs="+", default=[1.5, 2.0])
ap.add_argument("--c", type=int, nargs="+", default=[3, 4, 5, 6, 7, 8])
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
x = bench.make_volume(tuple(args.shape))
n = x.shape[0]
for m in args.m:
    for c in args.c:
        plan = pkg.FcmPlan(n, c, _lib.FCM_X_U8)
        plan.upload_pixels(x)
        plan.init_membership(0)
        plan.run(m, 1e-30, 2)  # warm-up (first launch configures the kernel)
        t = {}
        for k in (3, 7):
            ts = []
            for _ in range(args.reps):
                plan.init_membership(0)
                plan.run(m, 1e-30, k)
                ts.append(plan.timing()["loop_ms"])
            t[k] = float(np.median(ts))
        p = (t[7] - t[3]) / 4
        gbs = n * (1 + 8 * c) / (p * 1e-3) / 1e9
        print(f"m={m} c={c}: pass {p:.4f} ms  {gbs:7.1f} GB/s  ({n * (1 + 8 * c) / 1e9:.2f} GB/pass)", flush=True)
        plan.close()
