"""Where the end-to-end time of the public drop-in goes at a BASELINE config
(host phases of run_fcm_gpu and _iterate, wall clock, one GPU).

    python tools/e2e_phases.py [--config C4]
"""
import argparse
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
a = ap.parse_args()
shape, c, m, eps = bench.CONFIGS[a.config]
x8 = bench.make_volume(shape)
n = x8.shape[0]
x = x8.astype(np.float64)
cfg = pkg.FcmConfig(c=c, m=m, epsilon=eps, seed=0)


def t(label, fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    print(f"{label:48s} {1e3 * min(ts):9.2f} ms (min of {reps})", flush=True)
    return out


t("pixel_kind (float64 -> uint8, library, all cores)", lambda: pkg.pixel_kind(x))
plan = pkg.FcmPlan(n, c, _lib.FCM_X_U8)
t("upload_pixels (uint8, pageable)", lambda: plan.upload_pixels(x8))
plan.init_membership(0)
t("run (device seeded start + solve)", lambda: plan.run(m, eps, 500))
t("download_table (epilogue + 7 KB + host expansion, fresh arrays)", lambda: plan.download_table(x8))
u_out = np.empty(n * c)
l_out = np.empty(n, dtype=np.int32)
t("download_table (into reused arrays)", lambda: plan.download_table(x8, u_out=u_out, labels_out=l_out))
t("np.empty + first touch of n*c doubles", lambda: np.empty(n * c).fill(0.0))
u0 = pkg.init_membership(n, cfg).u
t("upload_membership (n*c doubles, pageable)", lambda: plan.upload_membership(u0))
t("run (uploaded start: prologue kernel + solve)", lambda: plan.run(m, eps, 500))
plan.close()
img = pkg.GrayImage(shape[2], shape[1] * shape[0], x)
t("run_fcm_gpu (whole call)", lambda: pkg.run_fcm_gpu(img, cfg))
t("_iterate(x, u0, cfg) (whole call)", lambda: pkg._iterate(x, u0.copy(), cfg))
