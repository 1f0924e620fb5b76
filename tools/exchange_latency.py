"""In-kernel root exchange of the multi-shard loop kernel, timed on one GPU.

    python tools/exchange_latency.py [C2|C4] [--shards 2 4 8]

One process, one B200: a plan with k shards on the same device runs k
cooperative loop kernels (each on its share of the SMs) that exchange their
2c+2-double rank roots every pass through the peer mailboxes
(fcm_tma_tree.cuh::exchange_roots) exactly as ranks on k GPUs do over NVLink.
With FCM_OPT_PROFILE each shard stamps its publication time into its mailbox
slot; shard 0's CTAs record when every root of the pass has arrived.  All
kernels read the same %globaltimer, so

    exchange latency = (all roots visible at a shard-0 CTA) - (last publication)

is the pure hand-off cost (system-scope release store -> acquire poll), free
of the shards' skew; the wait (all roots visible - this shard's own root
ready) adds the skew.  Cross-GPU NVLink adds its own hop latency on top.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from paper_1601_00072_b200.phantom import make_config  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
shards = [2, 4, 8]
if "--shards" in sys.argv:
    i = sys.argv.index("--shards")
    shards = [int(v) for v in sys.argv[i + 1:] if v.isdigit()]
    args = [a for a in args if not a.isdigit()]
cfg = args[0] if args else "C2"
x = make_config(cfg).reshape(-1).astype(np.uint8)
print(f"{cfg}: n={x.shape[0]}, c=3, m=2, one B200 (shards share its SMs)")
print(f"{'shards':>6s} {'us/iter':>8s} {'exch p50 us':>11s} {'exch p90 us':>11s} {'wait p50 us':>11s} {'passes':>6s}")
for k in [1] + shards:
    with pkg.FcmPlan(x.shape[0], 3, _lib.FCM_X_U8, devices=[0] * k) as plan:
        plan.upload_pixels(x)
        plan.init_membership(0)
        for _ in range(5):
            plan.run(2.0, 1e-5, 500)
        t = plan.timing()
        v, trace, iters, conv = plan.run(2.0, 1e-5, 500)
        t = plan.timing()
        us_iter = t["loop_ms"] * 1e3 / iters
        if k == 1:
            print(f"{k:6d} {us_iter:8.2f} {'-':>11s} {'-':>11s} {'-':>11s} {iters:6d}")
            continue
        plan.set_option(_lib.FCM_OPT_PROFILE, 1)
        plan.run(2.0, 1e-5, 500)
        P = plan.profile().astype(np.int64)
    ex, wt = [], []
    for it in range(1, P.shape[0] - 1):
        t_all, t_pub, t_root = P[it, :, 21], P[it, :, 22], P[it, :, 10]
        ok = (t_all > 0) & (t_pub > 0)
        if ok.any():
            ex.extend(((t_all - t_pub)[ok] / 1e3).tolist())
            wt.extend(((t_all - t_root)[ok & (t_root > 0)] / 1e3).tolist())
    ex, wt = np.array(ex), np.array(wt)
    print(f"{k:6d} {us_iter:8.2f} {np.median(ex):11.2f} {np.percentile(ex, 90):11.2f} {np.median(wt):11.2f} {iters:6d}")
