"""Stress the persistent loop kernel: many solves over many shapes, every result
must repeat bit for bit and no run may hit the in-kernel timeouts.

    python tools/stress.py [--minutes 4]
"""
import argparse
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from conftest import mixture_pixels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--minutes", type=float, default=4.0)
args = ap.parse_args()
rng = np.random.default_rng(2024)
t_end = time.time() + 60 * args.minutes
solves = cases = 0
while time.time() < t_end:
    n = int(rng.choice([3, 64, 1000, 39277, 200_003, 1_000_003, 7_109_137, 25_000_003]))
    c = int(rng.choice([2, 3, 4, 5, 8, 16])) if n >= 16 else 2
    m = float(rng.choice([1.5, 2.0, 2.0, 3.0]))
    shards = int(rng.choice([1, 1, 1, 2, 4]))
    x = np.clip(np.rint(mixture_pixels(n, c, seed=int(rng.integers(1 << 30)))), 0, 255).astype(np.uint8)
    devs = [0] * shards
    print(f"case n={n} c={c} m={m} shards={shards}", flush=True)
    with pkg.FcmPlan(n, c, _lib.FCM_X_U8, devices=devs) as plan:
        plan.upload_pixels(x)
        plan.init_membership(int(rng.integers(1 << 40)))
        first = None
        for rep in range(int(rng.integers(2, 6))):
            try:
                v, tr, k, conv = plan.run(m, 1e-5, 200)
            except pkg.DegenerateClusterError:
                first = first or "dead"
                break
            except pkg.FcmError as e:
                print("FAILED", n, c, m, shards, rep, plan.info(), e, flush=True)
                sys.exit(2)
            key = (v.tobytes(), tr.tobytes(), k, conv)
            if first is None:
                first = key
            elif key != first:
                print("NONDETERMINISTIC", n, c, m, shards, flush=True)
                sys.exit(1)
            solves += 1
        if first not in (None, "dead") and n <= 1_000_003 and rng.random() < 0.5:
            # table download == per-voxel download, bit for bit
            u0, l0 = plan.download()
            u1, l1 = plan.download_table(x, threads=int(rng.integers(0, 5)))
            if u0.tobytes() != u1.tobytes() or not np.array_equal(l0, l1):
                print("TABLE DOWNLOAD MISMATCH", n, c, m, shards, flush=True)
                sys.exit(3)
    cases += 1
print(f"stress ok: {cases} cases, {solves} solves", flush=True)
