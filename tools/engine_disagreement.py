"""How far apart are the reference's OWN two engines (sequential core._iterate
vs block-parallel parallel._iterate) on a BASELINE volume?  Both are fp64 and
differ only in summation order; their per-iteration objective-trace and
center disagreement is the yardstick for the GPU parity tolerances
(the symmetric-saddle start amplifies summation-order
differences ~4x per iteration for the first iterations).

Uses the oracle (bit-identical to the reference engines, tests/test_oracle.py).
Test/measurement infrastructure only.

    python tools/engine_disagreement.py --config C2 [--out profiles/engine_disagreement_C2.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from oracle import oracle as O  # noqa: E402
from paper_1601_00072_b200.phantom import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--c", type=int, default=3)
ap.add_argument("--m", type=float, default=2.0)
ap.add_argument("--out", default=None)
a = ap.parse_args()
x = make_config(a.config).astype(np.float64)
n = x.shape[0]
u0 = O.fill_membership_random(n, a.c, 0)
rows = {}
for engine in ("parallel", "sequential"):
    t0 = time.perf_counter()
    v, u, k, trace, conv = O.iterate(x, u0, a.c, a.m, 1e-5, 500, engine)
    rows[engine] = dict(v=v, u=u, k=k, trace=trace, conv=conv, s=time.perf_counter() - t0)
    print(engine, k, v, round(rows[engine]["s"], 1), "s", flush=True)
p, s = rows["parallel"], rows["sequential"]
kk = min(p["k"], s["k"])
rel = np.abs(p["trace"][:kk] - s["trace"][:kk]) / np.abs(s["trace"][:kk])
out = {
    "config": a.config, "n_voxels": int(n), "c": a.c, "m": a.m, "epsilon": 1e-5,
    "iterations": {"parallel": int(p["k"]), "sequential": int(s["k"])},
    "trace_rel_diff_per_iteration": [float(t) for t in rel],
    "trace_max_rel": float(rel.max()),
    "centers_max_rel": float(np.max(np.abs(p["v"] - s["v"]) / np.abs(s["v"]))),
    "membership_max_abs": float(np.abs(p["u"] - s["u"]).max()),
    "seconds": {"parallel": p["s"], "sequential": s["s"]},
}
print(json.dumps(out, indent=1))
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
