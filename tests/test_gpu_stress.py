"""Randomised shapes through the persistent loop kernel (a short version of
tools/stress.py): every solve repeats bit for bit, multi-shard plans agree
with one shard, and no run trips the in-kernel timeouts."""

import numpy as np
import pytest

from conftest import mixture_pixels

import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import _lib

pytestmark = pytest.mark.gpu


def test_random_shapes_repeat_and_shard_invariance():
    rng = np.random.default_rng(99)
    for _ in range(24):
        n = int(rng.choice([5, 777, 39277, 123_457, 1_000_003, 3_300_001]))
        c = int(rng.choice([2, 3, 5, 8])) if n > 8 else 2
        m = float(rng.choice([1.5, 2.0, 3.0]))
        x = np.clip(np.rint(mixture_pixels(n, c, seed=int(rng.integers(1 << 30)))), 0, 255).astype(np.uint8)
        seed = int(rng.integers(1 << 40))
        outs = []
        for devs in ([0], [0], [0, 0, 0, 0]):
            with pkg.FcmPlan(n, c, _lib.FCM_X_U8, devices=devs) as plan:
                plan.upload_pixels(x)
                plan.init_membership(seed)
                try:
                    v, tr, k, conv = plan.run(m, 1e-5, 150)
                except pkg.DegenerateClusterError as e:
                    outs.append(("dead", e.cluster))
                    continue
                _, lab = plan.download(membership=False)
                outs.append((v.tobytes(), tr.tobytes(), k, conv, lab.tobytes()))
        assert outs[0] == outs[1] == outs[2], (n, c, m)
