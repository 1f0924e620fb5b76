"""Phase breakdown of the loop kernel's passes (FCM_OPT_PROFILE timeline),
one GPU: for every probe, the median / max over CTAs of its offset from the
pass start (the earliest CTA's), averaged over passes 2..k-1.

    python tools/pass_phases.py C1 C3@1000000 C2 [--warm 20]

Probes (fcm_tma_*.cuh): 0 pass start, 13 consumers enter the stream (LUT
built), 12 first stage ready, 19 end-of-pass marker seen, 2 consumers done, 15 reducer drained its slots,
1 producer done claiming, 3 grid barrier released, 16 upper levels start,
17 level 1 from the tile partials done, 10 upper levels done, 14 finalize done.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1601_00072_b200 as pkg  # noqa: E402
from paper_1601_00072_b200 import _lib  # noqa: E402
from paper_1601_00072_b200.phantom import make_config  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
warm = 20
if "--warm" in sys.argv:
    warm = int(sys.argv[sys.argv.index("--warm") + 1])
    args.remove(str(warm))
PROBES = [(0, "start"), (13, "lut built"), (12, "1st stage"), (19, "end marker seen"),
          (2, "consumers done"), (15, "reducer done"),
          (1, "producer done"), (3, "barrier out"), (16, "upper start"), (17, "L1 done"), (10, "upper done"),
          (14, "finalize")]
for name in args or ["C1", "C2"]:
    x = make_config(name).reshape(-1)
    with pkg.FcmPlan(x.shape[0], 3, _lib.FCM_X_U8) as plan:
        plan.upload_pixels(x)
        plan.init_membership(0)
        for _ in range(warm):
            plan.run(2.0, 1e-5, 500)
        t_plain = plan.timing()["loop_ms"]
        plan.set_option(_lib.FCM_OPT_PROFILE, 1)
        v, trace, k, conv = plan.run(2.0, 1e-5, 500)
        t = plan.timing()
        P = plan.profile().astype(np.int64)
        info = plan.info()
    G = P.shape[1]
    print(f"\n{name}: n={x.shape[0]} tiles={info['tiles_local']} tile={info['tile']} grid={G} iters={k} "
          f"solve {t_plain * 1e3 / k:.2f} us/iter unprofiled ({t['loop_ms'] * 1e3 / k:.2f} profiled)")
    rows = []
    for it in range(1, min(k, P.shape[0]) - 1):
        t0 = P[it, :, 0].min()
        nxt = P[it + 1, :, 0].min() - t0
        row = []
        for slot, _ in PROBES:
            d = P[it, :, slot] - t0
            d = d[P[it, :, slot] > 0]
            row.append((np.median(d) / 1e3 if d.size else np.nan, d.max() / 1e3 if d.size else np.nan))
        rows.append((row, nxt / 1e3))
    med = np.nanmean([[r[0] for r in row] for row, _ in rows], axis=0)
    mx = np.nanmean([[r[1] for r in row] for row, _ in rows], axis=0)
    print(f"{'probe':18s} {'median us':>10s} {'max us':>8s}")
    for (slot, label), a, b in zip(PROBES, med, mx):
        print(f"{label:18s} {a:10.2f} {b:8.2f}")
    print(f"{'next pass start':18s} {np.mean([n for _, n in rows]):10.2f}")
