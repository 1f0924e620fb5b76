"""Device-side metrics and the CLI on a B200."""

import numpy as np
import pytest

from conftest import mixture_pixels

import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import cli, imgio, metrics
from paper_1601_00072_b200.phantom import make_config
from paper_1601_00072_b200.types import GrayImage, LabelMap

pytestmark = pytest.mark.gpu


def test_confusion_and_overlaps_vs_host():
    x = mixture_pixels(300_001, 4, seed=3)
    img = GrayImage(300_001, 1, x)
    res, plan = pkg.run_fcm_gpu(img, pkg.FcmConfig(c=4, m=2.0, epsilon=1e-5), keep_plan=True)
    with plan:
        rng = np.random.default_rng(1)
        ref = rng.integers(0, 3, size=x.shape[0]).astype(np.int32)
        conf = plan.confusion(ref, 3)
        host = np.bincount(res.labels.labels.astype(np.int64) * 3 + ref, minlength=12).reshape(4, 3)
        assert np.array_equal(conf, host)
        mask = rng.random(x.shape[0]) < 0.3
        counts, total = plan.mask_overlap(mask)
        assert total == int(mask.sum())
        assert np.array_equal(counts, np.bincount(res.labels.labels[mask], minlength=4))
        assert np.array_equal(plan.label_counts(), np.bincount(res.labels.labels, minlength=4))
        assert metrics.match_clusters_gpu(plan, LabelMap(300_001, 1, ref, 3), 4) == \
            metrics.match_clusters(res.labels, LabelMap(300_001, 1, ref, 3), 4)


def test_match_clusters_gpu_fewer_predicted_clusters():
    """plan.c < c: the device confusion is plan.c x c; the reference builds a
    c x c matrix whose extra prediction rows are zero (metrics.py:78-97)."""
    x = mixture_pixels(100_001, 3, seed=8)
    res, plan = pkg.run_fcm_gpu(GrayImage(100_001, 1, x), pkg.FcmConfig(c=3, m=2.0, epsilon=1e-5), keep_plan=True)
    with plan:
        ref = np.random.default_rng(2).integers(0, 4, size=x.shape[0]).astype(np.int32)
        want = metrics.match_clusters(res.labels, LabelMap(100_001, 1, ref, 4), 4)
        got = metrics.match_clusters_gpu(plan, LabelMap(100_001, 1, ref, 4), 4)
        assert len(got) == 4 and got == want


def test_pgm_raster_goes_straight_to_u8(tmp_path):
    x8 = make_config("C1")
    p = tmp_path / "c1.pgm"
    pkg.write_pgm(GrayImage(181, 217, x8.astype(np.float64)), p)
    raw = pkg.read_pgm_raster(p)
    assert raw.raster.dtype == np.uint8
    cfg = pkg.FcmConfig(c=3, m=2.0, epsilon=1e-5)
    a = pkg.run_fcm_gpu(raw, cfg)
    b = pkg.run_fcm_gpu(pkg.read_pgm(p), cfg)
    assert a.iterations == b.iterations and a.centers.v.tobytes() == b.centers.v.tobytes()
    assert a.membership.u.tobytes() == b.membership.u.tobytes()


def _truth_dir(tmp_path, labels, w, h):
    d = tmp_path / "truth"
    d.mkdir()
    for idx, name in enumerate(imgio.GROUND_TRUTH_CLASSES):
        pkg.write_pgm(GrayImage(w, h, (labels == idx).astype(np.float64) * 255.0), d / f"{name}.pgm")
    return d


def test_cli_segment_dsc_bench(tmp_path, capsys):
    # a 4-level phantom slice: tissue classes by intensity band, then noise
    rng = np.random.default_rng(5)
    w, h = 96, 80
    cls = rng.integers(0, 4, size=w * h)
    levels = np.array([215, 140, 70, 15])  # wm, gm, csf, background
    px = np.clip(levels[cls] + rng.integers(-6, 7, size=w * h), 0, 255)
    src = tmp_path / "in.pgm"
    pkg.write_pgm(GrayImage(w, h, px.astype(np.float64)), src)
    truth = _truth_dir(tmp_path, cls, w, h)
    out = tmp_path / "labels.pgm"
    assert cli.main(["segment", str(src), str(out), "-c", "4", "--epsilon", "1e-5", "--truth", str(truth)]) == 0
    seg_lines = capsys.readouterr().out.splitlines()
    assert cli.main(["dsc", str(out), str(truth), "-c", "4"]) == 0
    dsc_lines = capsys.readouterr().out.splitlines()
    # device-counted Dice == the reference flow over the written label map
    assert seg_lines[-4:] == dsc_lines and len(dsc_lines) == 4
    assert all(0.0 <= float(line.split()[1]) <= 1.0 for line in dsc_lines)
    csv_path = tmp_path / "t3.csv"
    assert cli.main(["bench", str(src), "--sizes", "8K,32K", "--runs", "2", "-c", "4", "--out", str(csv_path)]) == 0
    rows = open(csv_path).read().splitlines()
    assert rows[0] == "dataset_bytes,engine,run,seconds,iterations" and len(rows) == 5
    assert cli.main(["compare", str(src), "-c", "4", "--shards", "2"]) == 0
    cmp_lines = capsys.readouterr().out.splitlines()
    assert any("label agreement: 100.00%" in line for line in cmp_lines)
