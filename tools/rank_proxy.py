"""Per-rank pass of an N-GPU C4 solve, timed on ONE B200 (scaling proxy).

    python tools/rank_proxy.py [--passes 18]

For N in 1, 2, 4, 8: rank 0's plan of an N-rank job (fcm_plan_create_rank:
its octant-aligned slice of the 512^3 volume, the per-rank tree geometry)
runs its slice alone on this GPU (FCM_OPT_DEBUG_SOLO_RANK: everything a
rank's loop kernel does per pass except the root exchange).  A fixed number
of passes (epsilon 1e-300 never converges) isolates the steady pass:
(t(P) - t(2)) / (P - 2) from CUDA events around the loop kernel.  With the
exchange latency measured separately (tools/exchange_latency.py), the
N-GPU pass is estimated as t_rank(N) + t_exchange and the strong-scaling
factor as t_pass(1) / (t_rank(N) + t_exchange).  An estimate, not an N-GPU
measurement: each rank has a whole B200 here, which is exactly what it has
in an N-GPU job, but NVLink is not exercised.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from paper_1601_00072_b200.phantom import make_config  # noqa: E402

P = 18
if "--passes" in sys.argv:
    P = int(sys.argv[sys.argv.index("--passes") + 1])
exch = [float(v) for v in sys.argv[sys.argv.index("--exchange-us") + 1].split(",")] \
    if "--exchange-us" in sys.argv else None
x = make_config("C4").reshape(-1)
n = x.shape[0]


def steady_pass_ms(plan):
    def t(passes):
        ts = []
        for _ in range(7):
            plan.run(2.0, 1e-300, passes)
            ts.append(plan.timing()["loop_ms"])
        return float(np.median(ts[2:]))
    return (t(P) - t(2)) / (P - 2)


print(f"C4 {n} voxels, c=3, m=2; steady pass from {P} vs 2 passes (CUDA events, loop kernel)")
print(f"{'N':>2s} {'voxels/rank':>12s} {'tiles/rank':>10s} {'rank pass us':>12s} {'ideal us':>9s} {'eff':>5s}")
t1 = None
rows = []
for N in (1, 2, 4, 8):
    plan = pkg.FcmPlan.for_rank(n, 3, _lib.FCM_X_U8, 0, N, 0)
    try:
        if N > 1:
            plan.set_option(_lib.FCM_OPT_DEBUG_SOLO_RANK, 1)
        plan.upload_pixels(x[plan.voxel0:plan.voxel0 + plan.n_local])
        plan.init_membership(0)
        tp = steady_pass_ms(plan) * 1e3
        info = plan.info()
    finally:
        plan.close()
    if N == 1:
        t1 = tp
    rows.append((N, tp))
    print(f"{N:2d} {info['n_local']:12d} {info['tiles_local']:10d} {tp:12.2f} {t1 / N:9.2f} {t1 / N / tp:5.2f}")
if exch:
    print("\nestimated strong scaling with the measured exchange latency (us):")
    for (N, tp), e in zip(rows[1:], exch):
        print(f"  N={N}: pass {tp:.2f} + exchange {e:.2f} = {tp + e:.2f} us -> {t1 / (tp + e):.2f}x of 1 GPU")
