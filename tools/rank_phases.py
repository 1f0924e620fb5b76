"""Pass-phase timeline of rank 0 of an N-rank C4 job, run solo on one GPU
(FCM_OPT_DEBUG_SOLO_RANK; see tools/rank_proxy.py and tools/pass_phases.py).

    python tools/rank_phases.py [N]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from paper_1601_00072_b200.phantom import make_config  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
PROBES = [(0, "start"), (13, "lut built"), (12, "1st stage"), (19, "end marker seen"), (2, "consumers done"),
          (15, "reducer done"), (1, "producer done"), (3, "barrier arrive"), (16, "upper start"),
          (11, "level 2 done"), (10, "root done"), (14, "decided")]
x = make_config("C4").reshape(-1)
plan = pkg.FcmPlan.for_rank(x.shape[0], 3, _lib.FCM_X_U8, 0, N, 0)
if N > 1:
    plan.set_option(_lib.FCM_OPT_DEBUG_SOLO_RANK, 1)
plan.upload_pixels(x[plan.voxel0:plan.voxel0 + plan.n_local])
plan.init_membership(0)
for _ in range(5):
    plan.run(2.0, 1e-300, 18)
plan.set_option(_lib.FCM_OPT_PROFILE, 1)
plan.run(2.0, 1e-300, 18)
P = plan.profile().astype(np.int64)
info = plan.info()
plan.close()
print(f"rank 0 of {N}: n_local={info['n_local']} tiles={info['tiles_local']} grid={P.shape[1]}")
rows = []
for it in range(2, P.shape[0] - 1):
    t0 = P[it, :, 0].min()
    row = []
    for slot, _ in PROBES:
        d = P[it, :, slot] - t0
        d = d[P[it, :, slot] > 0]
        row.append((np.median(d) / 1e3 if d.size else np.nan, d.max() / 1e3 if d.size else np.nan))
    rows.append((row, (P[it + 1, :, 0].min() - t0) / 1e3))
med = np.nanmean([[r[0] for r in row] for row, _ in rows], axis=0)
mx = np.nanmean([[r[1] for r in row] for row, _ in rows], axis=0)
print(f"{'probe':18s} {'median us':>10s} {'max us':>8s}")
for (slot, label), a, b in zip(PROBES, med, mx):
    print(f"{label:18s} {a:10.2f} {b:8.2f}")
print(f"{'next pass start':18s} {np.mean([n for _, n in rows]):10.2f}")
