"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container only (it needs /root/reference and the reference
package built into oracle/_ref by oracle/build_ref.sh):

    python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/fcm_oracle.c) bit-for-bit against the
reference (tests/test_oracle.py) and give the GPU parity tests reference
outputs that travel to the GPU box (where /root/reference does not exist).

Inputs come from the reference's own test generators
(/root/reference/pkg/tests/conftest.py:9-67) and the SURVEY Appendix-A phantom.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)

import fcmseg  # noqa: E402  (the reference, compiled backend)
from fcmseg import _kernels as K  # noqa: E402
from fcmseg import core, parallel  # noqa: E402
from conftest import make_mixture_image, make_phantom, small_fixtures  # noqa: E402  (reference tests)

from paper_1601_00072_b200.phantom import phantom_slice  # noqa: E402

assert fcmseg.backend_name() == "compiled"


def kernels_fixture():
    out = {}
    # SplitMix64 streams (reference test_backends.py:23-40)
    for start, count in ((0, 3), (987654321, 100)):
        st, zs = start, []
        for _ in range(count):
            st, z = K.splitmix64(st)
            zs.append(z)
        out[f"splitmix_{start}"] = np.array(zs, dtype=np.uint64)
    # Seeded init for several shapes, including the full 64-bit seed range.
    for n, c, seed in ((257, 3, 77), (1000, 4, 7), (33, 8, 2**64 - 1), (5, 2, 424242), (1, 2, 0)):
        u = np.empty(n * c)
        K.fill_membership_random(u, n, c, seed)
        out[f"init_{n}_{c}_{seed}"] = u
    # Per-kernel outputs on the reference's TestKernelEquivalence input (test_backends.py:45-51).
    rng = np.random.default_rng(20)
    n, c = 257, 3
    x = np.rint(rng.random(n) * 255.0)
    u = np.empty(n * c)
    K.fill_membership_random(u, n, c, 77)
    v = np.array([12.0, 130.0, 244.0])
    out["k_x"], out["k_u"], out["k_v"] = x, u, v
    for m in (1.5, 2.0, 3.0):
        vv = np.empty(c)
        assert K.update_centers_linear(x, u, vv, n, c, m) == -1
        out[f"k_centers_m{m}"] = vv
        uu = np.empty(n * c)
        K.update_membership_range(x, v, uu, c, m, 0, n)
        out[f"k_memb_m{m}"] = uu
        out[f"k_obj_m{m}"] = np.array([K.objective_linear(x, u, v, n, c, m)])
    out["k_maxdiff"] = np.array([K.max_abs_diff(u, u[::-1].copy(), 0, n * c)])
    lab = np.empty(n, dtype=np.intc)
    K.argmax_rows(u, lab, n, c)
    out["k_argmax"] = lab.astype(np.int32)
    r2 = np.random.default_rng(21)
    for length in (1, 5, 16, 255, 1024, 1025):
        a = r2.random(length)
        nb = -(-length // 16)
        o = np.empty(nb)
        K.block_reduce_range(a, o, length, 8, 0, nb)
        out[f"br_in_{length}"] = a
        out[f"br_out_{length}"] = o
        out[f"br_sum_{length}"] = np.array([K.linear_sum(o, nb)])
    return out


def run_record(prefix, img_pixels, width, height, cfg, engine, out, keep_u=True):
    img = fcmseg.GrayImage(width, height, img_pixels)
    if engine == "sequential":
        res = core.run_fcm_sequential(img, cfg)
    else:
        res = parallel.run_fcm_parallel(img, cfg, workers=4)
    out[f"{prefix}_x"] = img.pixels
    out[f"{prefix}_cfg"] = np.array([cfg.c, cfg.m, cfg.epsilon, cfg.max_iters, cfg.seed], dtype=np.float64)
    out[f"{prefix}_v"] = res.centers.v
    out[f"{prefix}_labels"] = res.labels.labels.astype(np.int32)
    out[f"{prefix}_trace"] = np.array(res.objective_trace)
    out[f"{prefix}_iters"] = np.array([res.iterations])
    out[f"{prefix}_conv"] = np.array([int(res.converged)])
    if keep_u:
        out[f"{prefix}_u"] = res.membership.u


def runs_fixture():
    out = {}
    names = []
    # The reference's parity fixtures (conftest.small_fixtures, test_parallel.py:203-212).
    for idx, (img, cfg) in enumerate(small_fixtures(10)):
        for eng in ("sequential", "parallel"):
            p = f"small{idx}_{eng[:3]}"
            run_record(p, img.pixels, img.width, img.height, cfg, eng, out)
            names.append(p)
    # Reference fixture images (conftest.py:106-113) at several configs.
    ph = make_phantom(160, 128)
    mx = make_mixture_image(600, 3, seed=77, width=30)
    cases = [
        ("phantom_c4", ph, fcmseg.FcmConfig(c=4, m=2.0, epsilon=1e-5, seed=1)),
        ("phantom_c3_m3", ph, fcmseg.FcmConfig(c=3, m=3.0, epsilon=1e-5, seed=2)),
        ("phantom_c8_m15", ph, fcmseg.FcmConfig(c=8, m=1.5, epsilon=1e-5, seed=3)),
        ("mixture_c3", mx, fcmseg.FcmConfig(c=3, seed=77)),
        ("mixture_c2_m17", mx, fcmseg.FcmConfig(c=2, m=1.7, epsilon=1e-6, seed=9)),
        ("zero_c2", fcmseg.GrayImage(8, 1, np.zeros(8)), fcmseg.FcmConfig(c=2, seed=2)),
        ("twopop_c2", fcmseg.GrayImage(100, 1, np.array([10.0] * 50 + [200.0] * 50)),
         fcmseg.FcmConfig(c=2, seed=21)),
        ("cap1_c2", make_mixture_image(64, 2, seed=8), fcmseg.FcmConfig(c=2, seed=8, max_iters=1)),
    ]
    for p, img, cfg in cases:
        run_record(p, img.pixels, img.width, img.height, cfg, "sequential", out)
        names.append(p)
    # BASELINE config 1 (C1): the 181x217 slice, c=3, m=2, eps=1e-5, seed 0.
    c1 = phantom_slice(181, 217).reshape(-1).astype(np.float64)
    for p, cfg in (("C1", fcmseg.FcmConfig(c=3, m=2.0, epsilon=1e-5, seed=0)),
                   ("C1_c8_m15", fcmseg.FcmConfig(c=8, m=1.5, epsilon=1e-5, seed=0))):
        run_record(p, c1, 181, 217, cfg, "sequential", out, keep_u=True)
        names.append(p)
    out["names"] = np.array(names)
    return out


if __name__ == "__main__":
    k = kernels_fixture()
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **k)
    r = runs_fixture()
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **r)
    for f in ("kernels.npz", "runs.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
