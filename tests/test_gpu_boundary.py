"""GPU tests of the drop-in boundary's wider inputs and of the reference-side
registration:

* 16-bit pixels (FCM_X_U16, 2 B/voxel in HBM): the reference decodes 16-bit
  PGM samples (imgio.py:102-110) and accepts any finite intensity >= 0
  (types.py:38-41);
* 17 <= c <= 32 (the reference accepts any c >= 2, types.py:131);
* run_fcm_gpu registered inside the reference package itself
  (integration.register): `fcmseg segment --engine gpu` writes the same
  label PGM bytes as `--engine sequential` (the reference's own pin between
  its engines, tests/test_cli.py:43-51), and the reference's run_benchmark
  times the GPU engine through `_iterate` (bench.py:49-59);
* the per-thread plan cache of run_fcm_gpu / _iterate.
"""

import os
import sys

import numpy as np
import pytest

from conftest import REPO, mixture_pixels, run_case

import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import _lib

pytestmark = pytest.mark.gpu

CENTER_RTOL = 1e-9
U_ATOL = 1e-6


def _vs_oracle(x, c, m, eps, seed, width=None, height=1, trace_rtol=1e-9):
    from oracle import oracle as O
    n = x.shape[0]
    img = pkg.GrayImage(width or n, height, x.astype(np.float64))
    res = pkg.run_fcm_gpu(img, pkg.FcmConfig(c=c, m=m, epsilon=eps, max_iters=500, seed=seed))
    ref = O.run_fcm(x.astype(np.float64), c, m, eps, 500, seed)
    assert res.iterations == ref["iterations"] and res.converged == ref["converged"]
    assert np.allclose(res.centers.v, ref["centers"], rtol=CENTER_RTOL, atol=1e-12)
    assert np.abs(np.asarray(res.membership.u) - ref["membership"]).max() <= U_ATOL
    assert np.array_equal(np.asarray(res.labels.labels), ref["labels"])
    trel = np.abs(np.array(res.objective_trace) - ref["objective_trace"]) / np.abs(ref["objective_trace"])
    assert trel.max() <= trace_rtol, (trel.max(), int(trel.argmax()), trel)
    return res


def _u16_pixels(n, groups, seed):
    rng = np.random.default_rng(seed)
    levels = np.linspace(900, 60000, groups)
    return np.clip(rng.choice(levels, size=n) + rng.integers(-700, 701, size=n), 0, 65535).astype(np.uint16)


@pytest.mark.parametrize("c,m", [(3, 2.0), (4, 1.5), (5, 3.0)])
def test_uint16_pixels_vs_oracle(c, m):
    x = _u16_pixels(40_000, c, seed=c)
    assert pkg.pixel_kind(x.astype(np.float64))[0] == _lib.FCM_X_U16
    _vs_oracle(x, c, m, 1e-6, 5)


@pytest.mark.parametrize("c,m", [(3, 2.0), (8, 1.5)])
def test_uint16_loop_kernel_matches_per_pass_and_shards_bitwise(c, m):
    x = _u16_pixels(300_001, c, seed=11 + c)

    def solve(loop, devices=None):
        with pkg.FcmPlan(x.shape[0], c, _lib.FCM_X_U16, devices) as plan:
            plan.upload_pixels(x)
            plan.init_membership(7)
            plan.set_option(_lib.FCM_OPT_LOOP, loop)
            out = plan.run(m, 1e-5, 300)
            u, lab = plan.download()
        return out, u, lab

    (va, ta, ka, ca), ua, la = solve(1)
    for (vb, tb, kb, cb), ub, lb in (solve(0), solve(1, [0, 0, 0, 0])):
        assert ka == kb and ca == cb
        assert va.tobytes() == vb.tobytes() and ta.tobytes() == tb.tobytes()
        assert ua.tobytes() == ub.tobytes() and np.array_equal(la, lb)


def test_pgm16_raster_goes_straight_to_u16(tmp_path):
    """A 16-bit PGM (maxval > 255) reaches HBM at 2 B/voxel through
    read_pgm_raster, with the same result as the float64 GrayImage path."""
    x = _u16_pixels(96 * 64, 3, seed=9)
    path = tmp_path / "img16.pgm"
    pkg.write_pgm(pkg.GrayImage(96, 64, x.astype(np.float64)), path)
    raster = pkg.read_pgm_raster(path)
    assert raster.maxval > 255 and raster.raster.dtype == np.uint16
    cfg = pkg.FcmConfig(c=3, m=2.0, epsilon=1e-6, seed=4)
    a = pkg.run_fcm_gpu(raster, cfg)
    b = pkg.run_fcm_gpu(pkg.read_pgm(path), cfg)
    assert a.iterations == b.iterations
    assert a.centers.v.tobytes() == b.centers.v.tobytes()
    assert np.array_equal(a.labels.labels, b.labels.labels)


@pytest.mark.parametrize("c,m", [(17, 2.0), (24, 1.5), (32, 2.0)])
def test_more_than_16_clusters_vs_oracle(c, m):
    # c distinct, well-separated intensity groups so no cluster dies
    rng = np.random.default_rng(c)
    levels = np.linspace(3.0, 252.0, c)
    x = np.clip(np.rint(rng.choice(levels, size=6000) + rng.integers(-1, 2, size=6000)), 0, 255)
    # objective trace: with many clusters starting near the global mean (the
    # symmetric saddle of SURVEY.md 7) summation-order differences are
    # amplified for a few passes before the clusters separate.  The bar is
    # the reference's OWN disagreement between its two engines (sequential
    # vs block-parallel: same fp64 math, different summation order) on the
    # same input, x10, and never looser than 1e-9.
    from oracle import oracle as O
    for xx in (x, x + 0.5):  # integer pixels (uint8 path) and float64 pixels
        seq = O.run_fcm(xx, c, m, 1e-6, 500, 3)
        par = O.run_fcm(xx, c, m, 1e-6, 500, 3, engine="parallel")
        kk = min(seq["iterations"], par["iterations"])
        own = np.max(np.abs(seq["objective_trace"][:kk] - par["objective_trace"][:kk])
                     / np.abs(seq["objective_trace"][:kk]))
        _vs_oracle(xx, c, m, 1e-6, 3, trace_rtol=max(1e-9, 10.0 * own))


def test_more_than_16_clusters_shards_bitwise():
    x = np.clip(np.rint(mixture_pixels(200_003, 20, seed=20)), 0, 255).astype(np.uint8)

    def solve(devices):
        with pkg.FcmPlan(x.shape[0], 20, _lib.FCM_X_U8, devices) as plan:
            plan.upload_pixels(x)
            plan.init_membership(2)
            out = plan.run(2.0, 1e-5, 60)
            u, lab = plan.download()
        return out, u, lab

    (va, ta, ka, _), ua, la = solve(None)
    (vb, tb, kb, _), ub, lb = solve([0, 0])
    assert ka == kb and va.tobytes() == vb.tobytes() and ta.tobytes() == tb.tobytes()
    assert ua.tobytes() == ub.tobytes() and np.array_equal(la, lb)


def test_plan_cache_reuse_and_release():
    r = run_case("C1")
    img = pkg.GrayImage(181, 217, r["x"].astype(np.float64))
    cfg = pkg.FcmConfig(c=3, m=2.0, epsilon=1e-5, seed=0)
    a = pkg.run_fcm_gpu(img, cfg)
    b = pkg.run_fcm_gpu(img, cfg)  # same plan, fresh result arrays
    assert a.membership.u is not b.membership.u
    assert np.asarray(a.membership.u).tobytes() == np.asarray(b.membership.u).tobytes()
    other = pkg.run_fcm_gpu(img, pkg.FcmConfig(c=4, m=2.0, epsilon=1e-5, seed=0))  # new shape -> new plan
    assert other.centers.c == 4
    v, u, k, trace, conv = pkg._iterate(r["x"], None, cfg, seed=0)
    assert k == a.iterations and np.asarray(u).tobytes() == np.asarray(a.membership.u).tobytes()
    pkg.release_cached_plans()
    c = pkg.run_fcm_gpu(img, cfg)
    assert c.centers.v.tobytes() == a.centers.v.tobytes()


def _reference():
    ref = os.path.join(REPO, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "fcmseg")):
        pytest.skip("oracle/_ref (the installed reference) is absent")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import fcmseg
    return fcmseg


def test_reference_cli_segment_engine_gpu_writes_identical_bytes(tmp_path, capsys):
    """The reference's own `main(["segment", ..., "--engine", "gpu"])` with
    run_fcm_gpu registered: byte-identical label PGM to --engine sequential
    (reference tests/test_cli.py:43-51 pins sequential == parallel the same way)."""
    fcmseg = _reference()
    from fcmseg import cli, imgio, types
    from paper_1601_00072_b200.integration import register
    register(fcmseg)
    assert "gpu" in cli.ENGINES
    r = run_case("phantom_c4")  # the reference's test phantom (conftest.make_phantom), 160 x 128
    src = tmp_path / "phantom.pgm"
    imgio.write_pgm(types.GrayImage(160, 128, r["x"].astype(np.float64)), src)
    outs = {}
    for engine in ("sequential", "gpu"):
        outs[engine] = tmp_path / f"{engine}.pgm"
        assert cli.main(["segment", "--clusters", "4", "--seed", "3", "--engine", engine,
                         str(src), str(outs[engine])]) == 0
    printed = capsys.readouterr().out
    assert "engine: gpu" in printed
    assert outs["gpu"].read_bytes() == outs["sequential"].read_bytes()


def test_reference_run_benchmark_times_gpu_engine(tmp_path):
    """The reference's run_benchmark / write_csv with "gpu" registered: the GPU
    engine is timed through _iterate like the CPU engines (bench.py:49-59)
    and reports the same iteration counts."""
    fcmseg = _reference()
    from fcmseg import bench, types
    from paper_1601_00072_b200.integration import register
    register(fcmseg)
    r = run_case("C1")
    img = types.GrayImage(181, 217, r["x"].astype(np.float64))
    cfg = types.FcmConfig(c=3, m=2.0, epsilon=1e-5, seed=0)
    records, _ = bench.run_benchmark(img, [40_000, 80_000], runs=2, cfg=cfg, workers=2)
    by = {(rec.dataset_bytes, rec.engine): rec for rec in records}
    for size in {rec.dataset_bytes for rec in records}:
        assert by[(size, "gpu")].iterations == by[(size, "sequential")].iterations
        # (the first GPU run of a process also pays the CUDA context / module load)
        assert min(by[(size, "gpu")].seconds) < min(by[(size, "sequential")].seconds)
    out = tmp_path / "bench.csv"
    bench.write_csv(records, out)
    assert sum(1 for line in out.read_text().splitlines() if ",gpu," in line) == 4


def test_register_staged_kernel_only_above_16_clusters():
    """FCM_OPT_KERNEL = 1 (register-staged pass kernel) is the kernel of
    17 <= c <= 32 only: it lost its A/B against the TMA pipeline for c <= 16
    and is not built there, so a c <= 16 plan rejects it by name."""
    from paper_1601_00072_b200 import _lib
    with pkg.FcmPlan(10_000, 3, _lib.FCM_X_U8) as plan:
        with pytest.raises(pkg.InvalidConfigError, match="c > 16"):
            plan.set_option(_lib.FCM_OPT_KERNEL, 1)
    with pkg.FcmPlan(10_000, 20, _lib.FCM_X_U8) as plan:
        plan.set_option(_lib.FCM_OPT_KERNEL, 1)
