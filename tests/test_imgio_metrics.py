"""PGM I/O, metrics and CLI helpers of the drop-in (host side, no GPU).

Known answers mirror the reference's tests (test_imgio.py:26-125,
test_metrics.py:29-165); differential checks run against the reference
itself (oracle/_ref, built by oracle/build_ref.sh) when it is importable.
"""

import os
import sys

import numpy as np
import pytest

from conftest import REPO

import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import cli, imgio, metrics
from paper_1601_00072_b200.types import GrayImage, LabelMap


def _reference():
    path = os.path.join(REPO, "oracle", "_ref")
    if not os.path.isdir(os.path.join(path, "fcmseg")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import fcmseg
        return fcmseg
    except Exception:
        return None


class TestPgm:
    def test_ascii_and_binary(self):
        a = pkg.parse_pgm(b"P2\n2 2\n255\n0 10 20 30\n")
        b = pkg.parse_pgm(b"P5\n2 2\n255\n" + bytes([0, 10, 20, 30]))
        assert a.raster.dtype == np.uint8 and a.raster.tolist() == [0, 10, 20, 30]
        assert b.raster.tolist() == a.raster.tolist() and (b.width, b.height) == (2, 2)

    def test_comments_anywhere(self):
        img = pkg.parse_pgm(b"P2\n# made by hand\n2 1 # inline\n# another\n255\n5 # mid\n6\n")
        assert img.raster.tolist() == [5, 6]

    def test_sixteen_bit_big_endian(self):
        img = pkg.parse_pgm(b"P5\n2 1\n65535\n" + bytes([0x01, 0x02, 0xFF, 0xFE]))
        assert img.raster.dtype == np.uint16 and img.raster.tolist() == [258, 65534]

    def test_errors(self):
        with pytest.raises(pkg.UnsupportedMagicError):
            pkg.parse_pgm(b"P6\n1 1\n255\n\x00\x00\x00")
        with pytest.raises(pkg.MalformedHeaderError):
            pkg.parse_pgm(b"P2\nnot a number\n")
        with pytest.raises(pkg.MalformedHeaderError):
            pkg.parse_pgm(b"P2\n2 2\n70000\n0 0 0 0\n")
        with pytest.raises(pkg.TruncatedRasterError):
            pkg.parse_pgm(b"P5\n2 2\n255\n\x00\x01")
        with pytest.raises(pkg.TruncatedRasterError):
            pkg.parse_pgm(b"P2\n2 2\n255\n1 2 3\n")
        with pytest.raises(pkg.PgmValueError):
            pkg.parse_pgm(b"P2\n2 1\n100\n5 101\n")
        assert issubclass(pkg.TruncatedRasterError, pkg.PgmError) and issubclass(pkg.PgmError, ValueError)

    def test_round_trips(self, tmp_path):
        rng = np.random.default_rng(3)
        for maxval in (255, 65535):
            px = rng.integers(0, maxval + 1, size=6 * 7).astype(np.float64)
            p = tmp_path / f"r{maxval}.pgm"
            pkg.write_pgm(GrayImage(6, 7, px), p)
            back = pkg.read_pgm(p)
            assert back.pixels.tolist() == px.tolist() and (back.width, back.height) == (6, 7)
            raw = pkg.read_pgm_raster(p)
            assert raw.maxval == (255 if px.max() <= 255 else 65535)

    def test_label_levels(self, tmp_path):
        p = tmp_path / "l.pgm"
        pkg.write_pgm(LabelMap(4, 1, np.array([0, 1, 2, 3]), 4), p)
        assert pkg.read_pgm_raster(p).raster.tolist() == [0, 85, 170, 255]
        assert [pkg.label_intensity(j, 2) for j in range(2)] == [0, 255]
        with pytest.raises(ValueError):
            pkg.write_pgm(GrayImage(2, 1, np.array([1.5, 2.0])), p)

    def test_ground_truth(self, tmp_path):
        for name in imgio.GROUND_TRUTH_CLASSES:
            bits = np.zeros(6, dtype=np.uint8)
            bits[imgio.GROUND_TRUTH_CLASSES.index(name)] = 200
            pkg.write_pgm(GrayImage(3, 2, bits.astype(np.float64)), tmp_path / f"{name}.pgm")
        masks = pkg.read_ground_truth(tmp_path)
        assert [masks[k].count for k in imgio.GROUND_TRUTH_CLASSES] == [1, 1, 1, 1]
        os.remove(tmp_path / "csf.pgm")
        with pytest.raises(pkg.MissingClassError):
            pkg.read_ground_truth(tmp_path)

    def test_matches_reference_parser(self):
        ref = _reference()
        if ref is None:
            pytest.skip("reference not built (oracle/build_ref.sh)")
        from fcmseg.imgio import parse_pgm as ref_parse
        rng = np.random.default_rng(7)
        for _ in range(50):
            w, h = int(rng.integers(1, 9)), int(rng.integers(1, 9))
            maxval = int(rng.choice([1, 7, 255, 256, 4095, 65535]))
            px = rng.integers(0, maxval + 1, size=w * h)
            if rng.random() < 0.5:
                data = f"P2\n# c\n{w} {h}\n{maxval}\n".encode() + " ".join(map(str, px)).encode() + b"\n"
            else:
                body = px.astype(">u2" if maxval > 255 else np.uint8).tobytes()
                data = f"P5\n{w} {h}\n{maxval}\n".encode() + body
            a, b = pkg.parse_pgm(data), ref_parse(data)
            assert (a.width, a.height, a.maxval) == (b.width, b.height, b.maxval)
            assert a.raster.astype(np.int64).tolist() == b.raster.astype(np.int64).tolist()


class TestMetrics:
    def test_dsc_known_answers(self):
        a = metrics.BinaryMask(4, 1, np.array([1, 1, 0, 0]))
        b = metrics.BinaryMask(4, 1, np.array([1, 0, 0, 0]))
        e = metrics.BinaryMask(4, 1, np.zeros(4))
        assert metrics.dsc(a, a) == 1.0 and metrics.dsc(e, e) == 1.0 and metrics.dsc(a, e) == 0.0
        assert metrics.dsc(a, b) == pytest.approx(2 / 3)
        with pytest.raises(pkg.DimensionMismatchError):
            metrics.dsc(a, metrics.BinaryMask(2, 2, np.zeros(4)))

    def test_match_clusters_vs_reference(self):
        ref = _reference()
        rng = np.random.default_rng(11)
        for c in (2, 3, 4, 6):
            for _ in range(20):
                p = LabelMap(50, 1, rng.integers(0, c, 50), c)
                q = LabelMap(50, 1, rng.integers(0, c, 50), c)
                perm = metrics.match_clusters(p, q, c)
                assert sorted(perm) == list(range(c))
                if ref is not None:
                    from fcmseg.metrics import match_clusters as rm
                    from fcmseg.types import LabelMap as RL
                    assert perm == rm(RL(50, 1, p.labels, c), RL(50, 1, q.labels, c), c)

    def test_identity_and_transposition(self):
        lab = LabelMap(4, 1, np.array([0, 1, 2, 3]), 4)
        swapped = LabelMap(4, 1, np.array([1, 0, 2, 3]), 4)
        assert metrics.match_clusters(lab, lab, 4) == (0, 1, 2, 3)
        assert metrics.match_clusters(lab, swapped, 4) == (1, 0, 2, 3)


class TestCliHelpers:
    def test_parse_sizes(self):
        assert cli.parse_sizes("40K, 1m,100") == [40 * 1024, 1048576, 100]
        with pytest.raises(pkg.FcmError):
            cli.parse_sizes(" , ")

    def test_enlarge_matches_reference_layout(self):
        ref = _reference()
        rng = np.random.default_rng(2)
        img = imgio.PgmImage(5, 3, 255, rng.integers(0, 256, 15))
        for target in (15, 16, 60, 61, 1000):
            big = cli.enlarge(img, target)
            assert big.pixel_count >= target and big.width % 5 == 0
            if ref is not None:
                rb = ref.enlarge_dataset(ref.GrayImage(5, 3, img.raster.astype(np.float64)), target)
                assert (big.width, big.height) == (rb.width, rb.height)
                assert big.raster.astype(np.float64).tolist() == rb.pixels.tolist()

    def test_parser_has_every_command(self):
        p = cli.build_parser()
        for cmd in ("segment", "dsc", "bench", "compare"):
            assert p.parse_args([cmd] + (["a", "b"] if cmd in ("segment", "dsc") else ["a"])
                                + (["--sizes", "1K", "--out", "o"] if cmd == "bench" else [])).command == cmd
