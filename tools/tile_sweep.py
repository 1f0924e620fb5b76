import os, sys, subprocess, json
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
sizes = {"C1": 39277, "C3-200K": 235662, "C3-1M": 1178310}
tiles = [int(t) for t in sys.argv[1].split(",")]
name = sys.argv[2]
import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import _lib
from paper_1601_00072_b200.phantom import make_config
c1 = make_config("C1")
reps = {"C1": 1, "C3-200K": 6, "C3-1M": 30}[name]
x = np.tile(c1.reshape(217, 181), (1, reps)).reshape(-1) if reps > 1 else c1
with pkg.FcmPlan(x.shape[0], 3, _lib.FCM_X_U8) as plan:
    plan.upload_pixels(x); plan.init_membership(0)
    for _ in range(3): plan.run(2.0, 1e-5, 500)
    ts = []
    for _ in range(20):
        _, _, k, _ = plan.run(2.0, 1e-5, 500); ts.append(plan.timing()["loop_ms"])
    print(name, os.environ.get("FCM_TILE_EXPERIMENT"), x.shape[0], k, round(np.median(ts) * 1e3 / k, 2), "us/iter", plan.info()["tiles"])
