"""Small solves for compute-sanitizer (memcheck / synccheck / racecheck /
initcheck): the C1 slice through every launch mode the product uses, and
one volume above kSmallTiles (the owner-path loop kernel that prefetches the
next pass's static tile, stopped by max_iters with a prefetch in flight).

    compute-sanitizer --tool memcheck python tools/sanitize.py

Each case prints its iteration count; the sanitizer prints its own summary.
(Under a sanitizer concurrent kernels are serialised, so the 4-shard loop
kernels cannot meet in the exchange: that case exercises the timeout ->
per-pass fallback of fcm_run.)
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from paper_1601_00072_b200.phantom import make_config  # noqa: E402

only = sys.argv[1:] or None
x8 = make_config("C1")
n = x8.shape[0]


def case(name, kind=_lib.FCM_X_U8, x=x8, c=3, m=2.0, devices=None, opts=(), table=True, max_iters=500):
    if only and name not in only:
        return
    with pkg.FcmPlan(x.shape[0], c, kind, devices) as plan:
        plan.upload_pixels(x)
        plan.init_membership(0)
        for k, v in opts:
            plan.set_option(k, v)
        v, tr, it, conv = plan.run(m, 1e-5, max_iters)
        t = plan.timing()
        if table and kind == _lib.FCM_X_U8:
            u, lab = plan.download_table(x)
        else:
            u, lab = plan.download()
        plan.label_counts()
    print(f"{name:28s} iters={it:3d} launches={int(t['passes_launched'])} fallbacks={int(t['loop_fallbacks'])} "
          f"v0={v[0]:.6f}", flush=True)


case("loop_kernel")
case("loop_kernel_m15_lut", m=1.5)
case("per_pass_graph", opts=((_lib.FCM_OPT_LOOP, 0),))
case("per_pass_host", opts=((_lib.FCM_OPT_LOOP, 0), (_lib.FCM_OPT_GRAPH, 0)))
case("prologue_kernel", opts=((_lib.FCM_OPT_SEED_PASS, 0),))
case("recompute", opts=((_lib.FCM_OPT_RECOMPUTE, 1),))
case("shards4", devices=[0, 0, 0, 0], opts=((_lib.FCM_OPT_PEER_TIMEOUT_MS, 2000),))
case("u16", kind=_lib.FCM_X_U16, x=(x8.astype(np.uint16) * 200))
case("f64", kind=_lib.FCM_X_F64, x=x8.astype(np.float64) + 0.5)
case("c20", c=20, max_iters=30)
if only and "large_owner" in only:  # (not in the default list: minutes under memcheck)
    case("large_owner", x=make_config("C3@9000000"), max_iters=3)
