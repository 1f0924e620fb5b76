"""Per-pass timeline of the persistent loop kernel (FCM_OPT_PROFILE), one GPU.

    python tools/loop_timeline.py [--config C2] [--l2 1]
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
ap.add_argument("--config", default="C2")
ap.add_argument("--l2", type=int, default=1)
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--warm", type=int, default=3, help="solves before the profiled one (steady state: ~40)")
args = ap.parse_args()
shape, c, m, eps = bench.CONFIGS[args.config]
x = bench.make_volume(shape)
plan = pkg.FcmPlan(x.shape[0], c, _lib.FCM_X_U8)
plan.upload_pixels(x)
plan.init_membership(0)
plan.set_option(_lib.FCM_OPT_L2, args.l2)
plan.set_option(_lib.FCM_OPT_KERNEL, args.kernel)
for _ in range(args.warm):
    plan.run(m, eps, 500)
plan.set_option(_lib.FCM_OPT_PROFILE, 1)
v, trace, k, conv = plan.run(m, eps, 500)
t = plan.timing()
P = plan.profile().astype(np.int64)
info = plan.info()
print(f"{args.config}: iters {k} loop pass_ms {t['pass_ms']:.4f} grid {P.shape[1]} tiles {info['tiles_local']} tile {info['tile']}")
t0 = P[0, :, 0].min()
print("pass | start spread | claims done (min/med/max) | consumers done (min/med/max) | release | tiles/CTA min-max")
for it in range(min(k, P.shape[0])):
    s, cl, cd, rel = (P[it, :, j] - t0 for j in range(4))
    print(f"{it+1:4d} | {s.min()/1e3:7.2f}-{s.max()/1e3:7.2f} | {cl.min()/1e3:7.2f} {np.median(cl)/1e3:7.2f} {cl.max()/1e3:7.2f} | "
          f"{cd.min()/1e3:7.2f} {np.median(cd)/1e3:7.2f} {cd.max()/1e3:7.2f} | {rel.max()/1e3:7.2f} | {P[it,:,4].min()}-{P[it,:,4].max()}")

it = 1
s, cl, cd, rel, nt, last, smid = (P[it, :, j] for j in (0, 1, 2, 3, 4, 5, 6))
base = s.min()
order = np.argsort(cd)
print("pass 2: slowest CTAs: cta sm tiles last_claim claims_done consumers_done")
for b in list(order[-8:]) + list(order[:3]):
    print(b, smid[b], nt[b], (last[b] - base) / 1e3, (cl[b] - base) / 1e3, (cd[b] - base) / 1e3)
# CTAs on the same SM as the slowest
sl = order[-1]
print("same SM as slowest:", [(int(b), int(nt[b]), (cd[b] - base) / 1e3) for b in np.where(smid == smid[sl])[0]])

print("reducer (pass 2): polls per CTA mean", P[1, :, 8].mean(), "L1 nodes mean/max", P[1, :, 9].mean(), P[1, :, 9].max())
lag = (P[1, :, 7].astype(np.int64) - P[1, :, 2].astype(np.int64)) / 1e3
print("reducer lag us (mean/max)", lag.mean(), lag.max(), "argmax CTA", int(np.argmax(lag)))
b0 = int(P[1, :, 0].min())
print("consumers done max", (int(P[1, :, 2].max()) - b0) / 1e3, "reducers done max", (int(P[1, :, 7].max()) - b0) / 1e3,
      "barrier released", (int(P[1, :, 3].max()) - b0) / 1e3, "root done max", (int(P[1, :, 14].max()) - b0) / 1e3,
      "next start max", (int(P[2, :, 0].max()) - b0) / 1e3)

def mn0(j, it=1):
    return (np.median(P[it, :, j].astype(np.int64)) - int(P[it, :, 0].min())) / 1e3

def mx(j, it=1):
    return (int(P[it, :, j].max()) - int(P[it, :, 0].min())) / 1e3
print("pass 2 upper (max/median over CTAs): start", mx(16), mn0(16), "step0", mx(17), mn0(17), "step1", mx(11), mn0(11))
print("pass 2 chain (max over CTAs, us from pass start): consumers", mx(2), "reducers", mx(7), "barrier", mx(3),
      "upper step1", mx(11), "upper done", mx(10), "finalize", mx(14), "next start", (int(P[2, :, 0].max()) - int(P[1, :, 0].min())) / 1e3)

def mn(j, it=1):
    return (np.median(P[it, :, j].astype(np.int64)) - int(P[it, :, 0].min())) / 1e3
print("pass 2 start (median over CTAs, us): consumers start", mn(13), "first stage", mn(12), "| max:", mx(13), mx(12))

b0 = int(P[1, :, 0].min())
red = P[1, :, 7].astype(np.int64) - b0
o = np.argsort(red)[-5:]
print("slowest reducers (cta, slots done, reducer done, consumers done, nodes, polls):")
for b in o:
    print(int(b), (int(P[1, b, 15]) - b0) / 1e3, red[b] / 1e3, (int(P[1, b, 2]) - b0) / 1e3, int(P[1, b, 9]), int(P[1, b, 8]))
