import sys, numpy as np
sys.path.insert(0, '.')
import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import _lib
from paper_1601_00072_b200.phantom import make_config
for name in ["C1", "C2", "C3@200000"]:
    x = make_config(name).reshape(-1).astype(np.uint8)
    def solve(delay, shared):
        with pkg.FcmPlan(x.shape[0], 3, _lib.FCM_X_U8) as plan:
            plan.upload_pixels(x); plan.init_membership(0)
            plan.set_option(_lib.FCM_OPT_DEBUG_DELAY, delay)
            plan.set_option(_lib.FCM_OPT_DEBUG_SHARED_PARTIALS, shared)
            try:
                v, tr, k, conv = plan.run(2.0, 1e-5, 500)
            except Exception as e:
                return ("ERR", str(e)[:120])
            t = plan.timing()
            return (v.tobytes(), tr[:k].tobytes(), k, round(t["loop_ms"], 3))
    base = solve(0, 0)
    for d, sh in ((100000, 0), (100000, 1), (0, 1)):
        for rep in range(3):
            r = solve(d, sh)
            same = r[:3] == base[:3]
            print(name, "delay", d, "shared", sh, "same" if same else "DIFF", r[2:] if r[0] != "ERR" else r, flush=True)
