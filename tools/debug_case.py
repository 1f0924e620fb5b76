"""Run one GPU solve (debug helper): python tools/debug_case.py n c m loop [kernel] [float]"""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from conftest import mixture_pixels  # noqa: E402

n, c, m, loop = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
kernel = int(sys.argv[5]) if len(sys.argv) > 5 else 0
x = np.clip(np.rint(mixture_pixels(n, c, seed=21 + c)), 0, 255).astype(np.uint8)
plan = pkg.FcmPlan(n, c, _lib.FCM_X_U8)
plan.upload_pixels(x)
plan.init_membership(7)
plan.set_option(_lib.FCM_OPT_LOOP, loop)
plan.set_option(_lib.FCM_OPT_KERNEL, kernel)
print(plan.info(), flush=True)
v, tr, k, conv = plan.run(m, 1e-5, 300)
print("ok", k, conv, v[:4], plan.timing(), flush=True)
