"""Tile-size sweep of the loop kernel on one GPU (round 2: fence-free pass end,
butterfly tile end): us per iteration for each (volume, tile) pair.

    python tools/tile_sweep2.py

FCM_TILE_EXPERIMENT forces the tile (plan geometry, A/B only).  Each case runs
in a subprocess so the variable is read at plan creation.
"""
import os
import subprocess
import sys

CASES = {"C3@40000": [1024, 2048], "C3@100000": [1024, 2048], "C3@200000": [1024, 2048, 4096],
         "C3@500000": [1024, 2048, 4096], "C3@1000000": [2048, 4096, 8192], "C2": [4096, 8192, 16384]}
CHILD = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import _lib
from paper_1601_00072_b200.phantom import make_config
x = make_config(sys.argv[1]).reshape(-1)
with pkg.FcmPlan(x.shape[0], 3, _lib.FCM_X_U8) as plan:
    plan.upload_pixels(x); plan.init_membership(0)
    for _ in range(5): plan.run(2.0, 1e-5, 500)
    ts = []
    for _ in range(20):
        _, _, k, _ = plan.run(2.0, 1e-5, 500); ts.append(plan.timing()["loop_ms"])
    print(sys.argv[1], os.environ.get("FCM_TILE_EXPERIMENT", "default"), x.shape[0], k,
          round(float(np.median(ts)) * 1e3 / k, 2), "us/iter", plan.info()["tiles"], "tiles", flush=True)
'''
for name, tiles in CASES.items():
    for t in [None] + tiles:
        env = dict(os.environ)
        if t:
            env["FCM_TILE_EXPERIMENT"] = str(t)
        subprocess.run([sys.executable, "-c", CHILD, name], env=env, check=False)
